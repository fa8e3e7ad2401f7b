/*
 * conv_oracle.c -- CPU reference ("oracle") for Eq. 1 of Li et al., ASPLOS'21
 * (arXiv 2101.09808).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2101_09808_b200/, libconv.so) never links,
 * imports or calls it, and it shares no code, header or constant with it.
 *
 * What it computes (Sec. 1, Eq. 1):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,h+r,w+s] * Ker[k,c,r,s]
 *
 * stride 1, no padding (readings R2/R3), In NCHW with input extents
 * (H+R-1) x (W+S-1), Ker KCRS, Out NCHW with OUTPUT extents H x W (reading R1:
 * H, W are the loop extents N_h, N_w of Listing 2).
 *
 * Loop order is Listing 2's: n, k, c, r, s, h, w with
 * "Out +=" into a zeroed accumulator.  Accumulation is in double: every
 * product of two fp32 values is exact in double (24+24 <= 53 mantissa bits),
 * so the only rounding is the double summation, <= C*R*S * 2^-53 relative.
 * Parallelism (OpenMP) is over the (n,k) output planes only -- a
 * non-reduction split (Sec. 7) -- and each plane is summed
 * serially in Listing-2 order, so the result is independent of the thread
 * count.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Returns 0 on success, 1 if an extent is < 1 or a pointer is NULL. */
int oracle_conv_eq1(int N, int K, int C, int H, int W, int R, int S,
                    const float* in, const float* ker, double* out, int nthreads)
{
    if (N < 1 || K < 1 || C < 1 || H < 1 || W < 1 || R < 1 || S < 1) return 1;
    if (!in || !ker || !out) return 1;
    const int64_t Hin = (int64_t)H + R - 1;
    const int64_t Win = (int64_t)W + S - 1;
    const int64_t planes = (int64_t)N * K;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t nk = 0; nk < planes; ++nk) {
        const int64_t n = nk / K;
        const int64_t k = nk % K;
        double* acc = out + nk * (int64_t)H * W;           /* Out[n][k][:][:] */
        for (int64_t i = 0; i < (int64_t)H * W; ++i) acc[i] = 0.0;
        for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r)
                for (int64_t s = 0; s < S; ++s) {
                    const double kv = (double)ker[((k * C + c) * R + r) * S + s];
                    const float* in_rs = in + ((n * C + c) * Hin + r) * Win + s;
                    for (int64_t h = 0; h < H; ++h)
                        for (int64_t w = 0; w < W; ++w)
                            acc[h * W + w] += (double)in_rs[h * Win + w] * kv;
                }
    }
    return 0;
}

/*
 * Strided Eq. 1 (the paper's footnote: "we do not show
 * stride/dilation, but the methodology is applicable to the general case";
 * Table 1, marks the stride-2 layers with *):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+r,U*w+s] * Ker[k,c,r,s]
 *
 * In [N][C][Hin][Win] with explicit INPUT extents (Table 1 lists input
 * sizes), Out [N][K][H][W] with H = (Hin-R)/U + 1, W = (Win-S)/U + 1 (floor:
 * input rows/columns past the last full window are not read).  Same
 * Listing-2 loop order, double accumulation and (n,k)-plane parallelism as
 * oracle_conv_eq1.  Returns 0, or 1 on a bad extent / NULL pointer.
 */
int oracle_conv_eq1_strided(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                            const float* in, const float* ker, double* out, int nthreads)
{
    if (N < 1 || K < 1 || C < 1 || R < 1 || S < 1 || U < 1 || Hin < R || Win < S) return 1;
    if (!in || !ker || !out) return 1;
    const int64_t H = ((int64_t)Hin - R) / U + 1;
    const int64_t W = ((int64_t)Win - S) / U + 1;
    const int64_t planes = (int64_t)N * K;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t nk = 0; nk < planes; ++nk) {
        const int64_t n = nk / K;
        const int64_t k = nk % K;
        double* acc = out + nk * H * W;                    /* Out[n][k][:][:] */
        for (int64_t i = 0; i < H * W; ++i) acc[i] = 0.0;
        for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r)
                for (int64_t s = 0; s < S; ++s) {
                    const double kv = (double)ker[((k * C + c) * R + r) * S + s];
                    const float* in_rs = in + ((n * C + c) * (int64_t)Hin + r) * Win + s;
                    for (int64_t h = 0; h < H; ++h)
                        for (int64_t w = 0; w < W; ++w)
                            acc[h * W + w] += (double)in_rs[(U * h) * (int64_t)Win + U * w] * kv;
                }
    }
    return 0;
}

/*
 * Strided and dilated Eq. 1 (PAPER.md:201 footnote: "we do not show
 * stride/dilation, but the methodology is applicable to the general case"):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+D*r,U*w+D*s] * Ker[k,c,r,s]
 *
 * In [N][C][Hin][Win], H = (Hin - D*(R-1) - 1)/U + 1 (floor), likewise W.
 * Same Listing-2 loop order, double accumulation and (n,k)-plane
 * parallelism as oracle_conv_eq1.  Returns 0, or 1 on a bad extent / NULL.
 */
int oracle_conv_eq1_dilated(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D,
                            const float* in, const float* ker, double* out, int nthreads)
{
    if (N < 1 || K < 1 || C < 1 || R < 1 || S < 1 || U < 1 || D < 1) return 1;
    if ((int64_t)Hin < (int64_t)D * (R - 1) + 1 || (int64_t)Win < (int64_t)D * (S - 1) + 1) return 1;
    if (!in || !ker || !out) return 1;
    const int64_t H = ((int64_t)Hin - (int64_t)D * (R - 1) - 1) / U + 1;
    const int64_t W = ((int64_t)Win - (int64_t)D * (S - 1) - 1) / U + 1;
    const int64_t planes = (int64_t)N * K;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t nk = 0; nk < planes; ++nk) {
        const int64_t n = nk / K;
        const int64_t k = nk % K;
        double* acc = out + nk * H * W;
        for (int64_t i = 0; i < H * W; ++i) acc[i] = 0.0;
        for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r)
                for (int64_t s = 0; s < S; ++s) {
                    const double kv = (double)ker[((k * C + c) * R + r) * S + s];
                    const float* in_rs = in + ((n * C + c) * (int64_t)Hin + D * r) * Win + D * s;
                    for (int64_t h = 0; h < H; ++h)
                        for (int64_t w = 0; w < W; ++w)
                            acc[h * W + w] += (double)in_rs[(U * h) * (int64_t)Win + U * w] * kv;
                }
    }
    return 0;
}

/*
 * Zero-padded ("same"-style) Eq. 1 with stride U and dilation D (SURVEY.md
 * Sec. 8(f) NEXT-2; the paper's Eq. 1 has no padding, reading R3):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+D*r-ph,U*w+D*s-pw] * Ker[k,c,r,s]
 *
 * where In[...] outside [0,Hin) x [0,Win) is zero (the term is skipped --
 * written as the definition, with the bounds test, not by copying In into a
 * padded buffer).  H = (Hin + 2*ph - D*(R-1) - 1)/U + 1 (floor), likewise W.
 * Same loop order, double accumulation and (n,k)-plane parallelism as
 * oracle_conv_eq1.  Returns 0, or 1 on a bad extent / NULL.
 */
int oracle_conv_eq1_padded(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D, int ph, int pw,
                           const float* in, const float* ker, double* out, int nthreads)
{
    if (N < 1 || K < 1 || C < 1 || R < 1 || S < 1 || U < 1 || D < 1 || ph < 0 || pw < 0 || Hin < 1 || Win < 1)
        return 1;
    if ((int64_t)Hin + 2 * (int64_t)ph < (int64_t)D * (R - 1) + 1 ||
        (int64_t)Win + 2 * (int64_t)pw < (int64_t)D * (S - 1) + 1) return 1;
    if (!in || !ker || !out) return 1;
    const int64_t H = ((int64_t)Hin + 2 * (int64_t)ph - (int64_t)D * (R - 1) - 1) / U + 1;
    const int64_t W = ((int64_t)Win + 2 * (int64_t)pw - (int64_t)D * (S - 1) - 1) / U + 1;
    const int64_t planes = (int64_t)N * K;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t nk = 0; nk < planes; ++nk) {
        const int64_t n = nk / K;
        const int64_t k = nk % K;
        double* acc = out + nk * H * W;
        for (int64_t i = 0; i < H * W; ++i) acc[i] = 0.0;
        for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r)
                for (int64_t s = 0; s < S; ++s) {
                    const double kv = (double)ker[((k * C + c) * R + r) * S + s];
                    const float* plane = in + (n * C + c) * (int64_t)Hin * Win;
                    for (int64_t h = 0; h < H; ++h) {
                        const int64_t ih = U * h + D * r - ph;
                        if (ih < 0 || ih >= Hin) continue;           /* zero padding */
                        for (int64_t w = 0; w < W; ++w) {
                            const int64_t iw = U * w + D * s - pw;
                            if (iw < 0 || iw >= Win) continue;
                            acc[h * W + w] += (double)plane[ih * Win + iw] * kv;
                        }
                    }
                }
    }
    return 0;
}

/* Number of OpenMP threads a parallel region would use (for reporting). */
int oracle_num_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int t = 1;
#pragma omp parallel
    {
#pragma omp single
        t = omp_get_num_threads();
    }
    return t;
#else
    (void)nthreads;
    return 1;
#endif
}

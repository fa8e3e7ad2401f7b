// repack.cu -- layout transforms of the tensor-core paths (SURVEY.md Sec. 8(a)
// rows a-2 / a-3).  The paper counts its own packing (Sec. 6)
// and "any time expended in internal layout transformations"
// in every measurement; conv_run launches these inside the timed region.
//
//   K1 ker: KCRS fp32 -> [K][R][S][Cp]   (c innermost = the GEMM K order of
//           the im2col A operand), channels C..Cp-1 zero.
//   K2 in : NCHW fp32 -> [N][Hin][Win][Cp] (NHWC; TMA im2col needs channels
//           innermost and 16-B aligned pixel strides), channels C..Cp-1 zero.
// Both run in ONE launch (repack_all).
//
// Element conversion: TF32 path rounds to nearest, ties away (cvt.rna.tf32),
// BF16 path rounds to nearest even (cvt.rn.bf16x2).  Both are memory-bound
// (roofline: bytes / HBM bandwidth).
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include <type_traits>

#include "internal.h"
#include "sm100.cuh"

namespace conv {

__device__ __forceinline__ float to_tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// RNE pack of two fp32 into bf16x2 (lo in the low half)
__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
    uint32_t v;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(hi), "f"(lo));
    return v;
}

template <bool BF16>
struct Elem;
template <>
struct Elem<false> {
    using T = float;
    __device__ static T cvt(float x) { return to_tf32_rna(x); }
};
template <>
struct Elem<true> {
    using T = __nv_bfloat16;
    __device__ static T cvt(float x) { return __float2bfloat16_rn(x); }
};

// One launch performs both layout transforms (PAPER.md:371 packing; the
// two are independent, so merging them removes a kernel boundary):
//   CTAs [0, n_ker)          K1: Ker KCRS fp32 -> [K][R][S][Cp], one CTA per
//                            (k, chunk of `cc` channels): the chunk's cc*R*S
//                            contiguous floats are staged in shared memory with
//                            coalesced loads, then written c-innermost with
//                            coalesced stores; channels C..Cp-1 are zero.
//   CTAs [n_ker, n_ker+n_in) K2: NCHW fp32 -> NHWC, one CTA per (image,
//                            64-channel block, 64-pixel block) through a padded
//                            64x65 tile: float4 loads along pixels (scalar when
//                            the pixel count is not a multiple of 4), 16-B
//                            stores of 8 bf16 / 4 fp32 consecutive channels.
struct RepackGeom {
    int C, Cp, RS, cc, ker_chunks;   // K1
    int K, krows;                    // K1: output channels; Ker rows per CTA (> 1 only if ker_chunks == 1)
    int64_t P;                       // K2: pixels per image
    int ptiles, ctiles;              // K2 tile grid per image
    int n_ker;                       // number of K1 CTAs
    int N;                           // images
    int64_t n_tiles;                 // K2 tiles (TMA variant)
    int pdl_from;                    // first block that triggers the dependent launch
    int* zero_ptr;                   // fused main kernel: reserved ints + chunk flags to clear
    int zero_n;                      //   (ints; spread over the K1 CTAs)
    int pre_q, pre_ch, nch;          // fused: prologue tiles (K2 CTAs for q < pre_q, channels
                                     //   [0, 64)) whose chunk flags the launch sets (not clears)
    int n_pre;                       // fused: number of prologue K2 CTAs (pre_q x 64-channel tiles)
    int cc_f;                        // fused: channels per chunk (flag column granularity)
};

// K1 for many short rows (whole rows fit, K >= 4 CTAs per SM): Ker rows
// [k0, k0 + krows) of one CTA are one contiguous KCRS slab of krows * C * RS
// fp32, staged in shared memory and written row by row as [RS][Cp]
// (channels >= C zero).  A separate function so that the common one-row
// path stays the short code path it was (its instructions are fetched cold
// after every L2 flush).
template <bool BF16, int NT>
__device__ __noinline__ void ker_repack_rows(const float* __restrict__ ker, typename Elem<BF16>::T* __restrict__ ker_ws,
                                             const RepackGeom g, float* sm) {
    const int tid = threadIdx.x;
    const int64_t k0 = (int64_t)blockIdx.x * g.krows;
    const int nrows = (int)min((int64_t)g.krows, g.K - k0);
    const int row_f = g.C * g.RS;                       // staged floats per row
    const float* src = ker + k0 * row_f;
    const int nld = nrows * row_f;
    if (((reinterpret_cast<uintptr_t>(src) | (uintptr_t)nld * 4) & 15) == 0) {
        // 16-B copies (the slab and its length are 16-B multiples): a quarter
        // of the instructions for the weight-heavy 1x1 layers (Y23: 116 MB)
        for (int i = tid * 4; i < nld; i += NT * 4) {
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm + i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + i) : "memory");
        }
    } else {
        for (int i = tid; i < nld; i += NT) {
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm + i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + i) : "memory");
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // (row, tap) output rows of Cp channels; bf16 pairs packed (Cp even)
    const int width = g.Cp;
    for (int rr = 0; rr < nrows * g.RS; ++rr) {
        const int r = rr / g.RS, rs = rr - r * g.RS;
        const float* sr = sm + r * row_f + rs;
        typename Elem<BF16>::T* d = ker_ws + ((k0 + r) * g.RS + rs) * (int64_t)g.Cp;
        if (BF16) {
            uint32_t* d2 = reinterpret_cast<uint32_t*>(d);
            for (int c2 = tid; c2 < (width >> 1); c2 += NT) {
                const int c = 2 * c2;
                d2[c2] = pack2_bf16(c < g.C ? sr[c * g.RS] : 0.0f, c + 1 < g.C ? sr[(c + 1) * g.RS] : 0.0f);
            }
        } else {
            for (int c = tid; c < width; c += NT) d[c] = Elem<BF16>::cvt(c < g.C ? sr[c * g.RS] : 0.0f);
        }
    }
}

// K1, one CTA (NT threads): Ker row k = blockIdx.x / ker_chunks, channels
// [c0, c0 + cc): stage the contiguous KCRS slice (cload * RS fp32) in shared
// memory, then write it as [RS][Cp] (channels >= C zero), converted.
template <bool BF16, int NT>
__device__ __forceinline__ void ker_repack_cta(const float* __restrict__ ker, typename Elem<BF16>::T* __restrict__ ker_ws,
                                               const RepackGeom& g, float* sm) {
    const int tid = threadIdx.x;
    if (g.krows > 1) {
        ker_repack_rows<BF16, NT>(ker, ker_ws, g, sm);
        return;
    }
    const int64_t k = blockIdx.x / g.ker_chunks;
    const int c0 = (blockIdx.x % g.ker_chunks) * g.cc;
    const int c1 = min(c0 + g.cc, g.Cp);
    const int cload = max(0, min(c1, g.C) - c0);
    const float* src = ker + (k * g.C + c0) * g.RS;
    // the whole slice in flight at once: asynchronous global -> shared copies
    // (register round trips, even eight deep, cap a weight-heavy repack at
    // ~2.5 TB/s); 16-B copies when the slice is 16-B aligned (cc is a
    // multiple of 4 channels)
    const int nld = cload * g.RS;
    const bool v16 = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)nld * 4) & 15) == 0;
    for (int i = v16 ? tid * 4 : tid; i < nld; i += v16 ? NT * 4 : NT) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm + i));
        if (v16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + i) : "memory");
        else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + i) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    typename Elem<BF16>::T* dst = ker_ws + k * (int64_t)g.RS * g.Cp;
    const int width = c1 - c0;
    // Wide slices: one output row (tap rs) at a time, channels across the
    // threads -- no per-element division (a division per element made the
    // weight-heavy repacks issue-bound at ~2.5 TB/s); bf16 pairs are packed
    // into one 4-B store (c0, width and Cp are even: the host keeps cc even).
    // Narrow slices (few channels, e.g. 3-channel 7x7 stems): the flattened
    // (tap, channel) loop keeps every thread busy.
    if (width < NT / 2) {
        for (int e = tid; e < g.RS * width; e += NT) {
            const int rs = e / width;
            const int c = e - rs * width;
            dst[(int64_t)rs * g.Cp + c0 + c] = Elem<BF16>::cvt(c0 + c < g.C ? sm[c * g.RS + rs] : 0.0f);
        }
    } else if (BF16 && !((c0 | width) & 1)) {
        const int hw = width >> 1;
        for (int rs = 0; rs < g.RS; ++rs) {
            uint32_t* d = reinterpret_cast<uint32_t*>(dst + (int64_t)rs * g.Cp + c0);
            for (int c2 = tid; c2 < hw; c2 += NT) {
                const int c = 2 * c2;
                const float lo = c0 + c < g.C ? sm[c * g.RS + rs] : 0.0f;
                const float hi = c0 + c + 1 < g.C ? sm[(c + 1) * g.RS + rs] : 0.0f;
                d[c2] = pack2_bf16(lo, hi);
            }
        }
    } else {
        for (int rs = 0; rs < g.RS; ++rs) {
            typename Elem<BF16>::T* d = dst + (int64_t)rs * g.Cp + c0;
            for (int c = tid; c < width; c += NT)
                d[c] = Elem<BF16>::cvt(c0 + c < g.C ? sm[c * g.RS + rs] : 0.0f);
        }
    }
}

// MODE 0: K1 + K2 (plain plans); 1: + clearing (split-K arrival counters);
// 2: K1 + clearing + the fused prologue (fused plans).  Separate instances:
// compiled into one kernel the untaken clearing / prologue code cost the
// plain repack ~1 % of the Table-1 sweep (its instructions are fetched cold
// after every L2 flush).
template <bool BF16, int MODE>
__global__ void __launch_bounds__(256) repack_all(const float* __restrict__ in, const float* __restrict__ ker,
                                                  typename Elem<BF16>::T* __restrict__ in_ws,
                                                  typename Elem<BF16>::T* __restrict__ ker_ws, const RepackGeom g) {
    extern __shared__ float sm[];
    const int tid = threadIdx.x;
    // Programmatic dependent launch: the main kernel (one 200-KB CTA per SM)
    // may start its prologue once every CTA of this grid has triggered or
    // exited.  Only the last wave triggers, so the main kernel does not take
    // SMs away from the bulk of the repack; it waits for this grid's
    // completion (griddepcontrol.wait) before reading the workspace.
    if ((int)blockIdx.x >= g.pdl_from) asm volatile("griddepcontrol.launch_dependents;");
    if ((int)blockIdx.x < g.n_ker) {
        // ---- K1 ----
        if (MODE >= 1 && g.zero_n) {   // clear the fused transform's chunk flags (the prologue's are set below)
            const int per = (g.zero_n + g.n_ker - 1) / g.n_ker;
            const int z0 = blockIdx.x * per, z1 = min(z0 + per, g.zero_n);
            for (int i = z0 + tid; i < z1; i += 256) {
                const int f = i - 32;   // flag index q * nch + ch
                const bool pre = f >= 0 && f / g.nch < g.pre_q && f % g.nch < g.pre_ch;
                if (!pre) g.zero_ptr[i] = 0;
            }
        }
        ker_repack_cta<BF16, 256>(ker, ker_ws, g, sm);
        return;
    }
    // ---- K2 ----
    float (*tile)[65] = reinterpret_cast<float (*)[65]>(sm);
    int b = blockIdx.x - g.n_ker;
    int pt, ct;
    int64_t n;
    const int pre_ct = (g.pre_ch * g.cc_f + 63) / 64;   // 64-channel tiles in the prologue
    if (MODE == 2 && g.n_pre) {                   // fused prologue: tile (q = b / pre_ct, channels 64 * (b % pre_ct) ...)
        ct = b % pre_ct;
        const int q = b / pre_ct;
        n = q / g.ptiles;
        pt = q % g.ptiles;
    } else {
        pt = b % g.ptiles;
        b /= g.ptiles;
        ct = b % g.ctiles;
        n = b / g.ctiles;
    }
    const int64_t P = g.P;
    const int C = g.C, Cp = g.Cp;
    const int64_t p0 = (int64_t)pt * 64;
    const int c0 = ct * 64;
    const float* src = in + n * C * P;
    if ((P & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * 256;
            const int cl = idx >> 4, pq = (idx & 15) * 4;
            const int c = c0 + cl;
            const int64_t p = p0 + pq;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < C && p < P) v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)c * P + p));
            tile[cl][pq] = v.x; tile[cl][pq + 1] = v.y; tile[cl][pq + 2] = v.z; tile[cl][pq + 3] = v.w;
        }
    } else {
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {
            const int idx = tid + i * 256;
            const int cl = idx >> 6, pl = idx & 63;
            const int c = c0 + cl;
            const int64_t p = p0 + pl;
            tile[cl][pl] = (c < C && p < P) ? __ldg(src + (int64_t)c * P + p) : 0.0f;
        }
    }
    __syncthreads();
    typename Elem<BF16>::T* dst = in_ws + n * P * Cp;
    constexpr int kVec = BF16 ? 8 : 4;               // channels per 16-B store
    constexpr int kChunks = 64 / kVec;               // 16-B chunks per pixel row of the tile
#pragma unroll
    for (int i = 0; i < (64 * kChunks) / 256; ++i) {
        const int idx = tid + i * 256;
        const int pl = idx / kChunks, cq = (idx % kChunks) * kVec;
        const int64_t p = p0 + pl;
        const int c = c0 + cq;
        if (p < P && c < Cp) {
            if (BF16) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const __nv_bfloat162 bb = __floats2bfloat162_rn(tile[cq + 2 * j][pl], tile[cq + 2 * j + 1][pl]);
                    w[j] = *reinterpret_cast<const uint32_t*>(&bb);
                }
                *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + p * Cp + c) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
                float4 v;
                v.x = to_tf32_rna(tile[cq][pl]);
                v.y = to_tf32_rna(tile[cq + 1][pl]);
                v.z = to_tf32_rna(tile[cq + 2][pl]);
                v.w = to_tf32_rna(tile[cq + 3][pl]);
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + p * Cp + c) = v;
            }
        }
    }
    // fused prologue: the main kernel reads these chunks only after this grid
    // has completed (griddepcontrol.wait), so plain stores suffice
    if (MODE == 2 && g.n_pre) {
        const int q = (blockIdx.x - g.n_ker) / pre_ct;
        const int ch0 = ct * 64 / g.cc_f, ch1 = min(ch0 + 64 / g.cc_f, g.pre_ch);
        if (tid < ch1 - ch0) g.zero_ptr[32 + (int64_t)q * g.nch + ch0 + tid] = 1;
    }
}

// K2 with TMA (used when the NCHW pixel stride P*4 is a multiple of 16 B):
// persistent CTAs of 128 threads loop over (image, 64-channel, 64-pixel)
// tiles.  A 3-D TMA load brings the [64 ch][64 px] fp32 box of NCHW into
// shared memory (channels >= C are zero-filled by the TMA: that is the Cp
// padding); the threads convert it into the 128B-swizzled [64 px][64 ch] box
// (bf16: one 128-B row per pixel; tf32: two 32-channel boxes) and one thread
// TMA-stores it into the NHWC workspace.  Loads and stores are double-
// buffered, so each SM keeps two 16-KB loads in flight with few instructions.
// CTAs [0, n_ker) run K1 exactly as in repack_all.
template <bool BF16>
__global__ void __launch_bounds__(128) repack_tma(const float* __restrict__ ker,
                                                  typename Elem<BF16>::T* __restrict__ ker_ws,
                                                  const __grid_constant__ CUtensorMap src_map,
                                                  const __grid_constant__ CUtensorMap dst_map, const RepackGeom g) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smraw[];
    const int tid = threadIdx.x;
    if ((int)blockIdx.x >= g.pdl_from) asm volatile("griddepcontrol.launch_dependents;");
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    if ((int)blockIdx.x < g.n_ker) {
        ker_repack_cta<BF16, 128>(ker, ker_ws, g, reinterpret_cast<float*>(sm));
        return;
    }
    float* in_buf[2] = {reinterpret_cast<float*>(sm), reinterpret_cast<float*>(sm + 16384)};
    uint8_t* out_buf[2] = {sm + 32768, sm + 49152};
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + 65536);
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t first = blockIdx.x - g.n_ker;
    const int64_t stride = gridDim.x - g.n_ker;
    auto coords = [&](int64_t tile, int& px, int& cx, int& n) {
        px = (int)(tile % g.ptiles) * 64;
        const int64_t t2 = tile / g.ptiles;
        cx = (int)(t2 % g.ctiles) * 64;
        n = (int)(t2 / g.ctiles);
    };
    if (tid == 0 && first < g.n_tiles) {
        int px, cx, n;
        coords(first, px, cx, n);
        mbar_arrive_expect_tx(&full[0], 16384);
        tma_load_3d(in_buf[0], &src_map, &full[0], px, cx, n);
    }
    int i = 0;
    for (int64_t tile = first; tile < g.n_tiles; tile += stride, ++i) {
        const int b = i & 1;
        const int64_t next = tile + stride;
        if (tid == 0 && next < g.n_tiles) {       // prefetch into the other buffer (released at barrier B)
            int px, cx, n;
            coords(next, px, cx, n);
            mbar_arrive_expect_tx(&full[b ^ 1], 16384);
            tma_load_3d(in_buf[b ^ 1], &src_map, &full[b ^ 1], px, cx, n);
        }
        mbar_wait(&full[b], (i >> 1) & 1);
        if (tid == 0) bulk_wait_read<1>();        // the store of tile i-2 has read out_buf[b]
        __syncthreads();                          // (A)
        const int p = tid & 63, half = tid >> 6;  // pixel, channel half
        const float* src = in_buf[b] + (half * 32) * 64 + p;
        if (BF16) {
            // row p = 64 channels x 2 B = 128 B; 16-B chunk j holds channels 8j..8j+7
            uint8_t* row = out_buf[b] + p * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = half * 4 + q;
                uint4 o;
                const float* s = src + (q * 8) * 64;
                o.x = pack2_bf16(s[0], s[64]);
                o.y = pack2_bf16(s[128], s[192]);
                o.z = pack2_bf16(s[256], s[320]);
                o.w = pack2_bf16(s[384], s[448]);
                *reinterpret_cast<uint4*>(row + ((j ^ (p & 7)) << 4)) = o;
            }
        } else {
            // box `half` (32 channels x 4 B = 128 B per pixel row); chunk j = 4 channels
            uint8_t* row = out_buf[b] + half * 8192 + p * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float* s = src + (j * 4) * 64;
                float4 o;
                o.x = to_tf32_rna(s[0]);
                o.y = to_tf32_rna(s[64]);
                o.z = to_tf32_rna(s[128]);
                o.w = to_tf32_rna(s[192]);
                *reinterpret_cast<float4*>(row + ((j ^ (p & 7)) << 4)) = o;
            }
        }
        fence_proxy_async_smem();
        __syncthreads();                          // (B) out_buf[b] written, in_buf[b] consumed
        if (tid == 0) {
            int px, cx, n;
            coords(tile, px, cx, n);
            tma_store_3d(&dst_map, out_buf[b], cx, px, n);
            if (!BF16) tma_store_3d(&dst_map, out_buf[b] + 8192, cx + 32, px, n);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait<0>();
}

cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev, bool with_in,
                          const RepackFuse& fz) {
    RepackGeom g;
    g.zero_ptr = fz.zero_ptr;
    g.zero_n = fz.zero_n;
    g.pre_q = fz.pre_q;
    g.pre_ch = fz.pre_ch;
    g.nch = fz.nch > 0 ? fz.nch : 1;
    g.cc_f = fz.cc > 0 ? fz.cc : 1;
    g.n_pre = (!with_in && fz.pre_ch > 0) ? fz.pre_q * ((fz.pre_ch * g.cc_f + 63) / 64) : 0;
    const int zero_n = fz.zero_n;
    g.C = pb.C;
    g.Cp = Cp;
    g.RS = pb.R * pb.S;
    // channels per K1 CTA so that the staged slice is <= 32 KB (at least 1)
    g.cc = std::max(1, std::min(Cp, (int)(32768 / (4 * g.RS))));
    if (g.cc > 4) g.cc &= ~3;          // multiple of 4: 16-B aligned slices (and even for bf16 pairs)
    else if (g.cc > 1) g.cc &= ~1;     // even: bf16 channel pairs share a 4-B store
    g.ker_chunks = (Cp + g.cc - 1) / g.cc;
    g.K = pb.K;
    // whole rows fit and there are many of them: several consecutive
    // (contiguous) rows per CTA, so that short rows (1x1 kernels: one 4-KB
    // row of C = 1024, K = 28269) do not make tens of thousands of tiny CTAs
    // -- but never fewer than ~4 CTAs per SM (a few long CTAs serialise:
    // measured 9 -> 23-32 us on the 128-row and 3-channel Table-1 layers)
    static int dev_sms = [] {
        int n = 148, d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
    }();
    g.krows = g.ker_chunks == 1
                  ? std::max(1, std::min(8192 / std::max(1, pb.C * g.RS), pb.K / (4 * dev_sms)))
                  : 1;
    g.n_ker = ((pb.K + g.krows - 1) / g.krows) * g.ker_chunks;
    g.P = pb.Hin() * pb.Win();
    g.ptiles = (int)((g.P + 63) / 64);
    g.ctiles = (Cp + 63) / 64;
    g.N = pb.N;
    g.n_tiles = (int64_t)g.ptiles * g.ctiles * pb.N;
    // The TMA variant measured slower than repack_all in r01 (27.5 vs 23.7 us,
    // batched bf16); kept for study behind CONV_TMA_REPACK=1.
    static const bool want_tma = getenv("CONV_TMA_REPACK") != nullptr;
    const bool use_tma = with_in && zero_n == 0 && want_tma && (g.P % 4 == 0) && g.cc * g.RS * 4 <= 32768 &&
                         g.n_tiles < (1ll << 31) && g.P < (1ll << 31);
    if (use_tma) {
        CUtensorMap src_map, dst_map;
        {
            cuuint64_t dims[3] = {(cuuint64_t)g.P, (cuuint64_t)pb.C, (cuuint64_t)pb.N};
            cuuint64_t strides[2] = {(cuuint64_t)g.P * 4, (cuuint64_t)g.P * 4 * pb.C};
            cuuint32_t box[3] = {64, 64, 1};
            cuuint32_t es[3] = {1, 1, 1};
            if (g_encode_tiled(&src_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return cudaErrorInvalidValue;
        }
        {
            const int es_b = bf16 ? 2 : 4;
            // 3-D {Cp, P, N}: boxes that run past the image's last pixel are
            // clipped at the image, never spill into the next one
            cuuint64_t dims[3] = {(cuuint64_t)Cp, (cuuint64_t)g.P, (cuuint64_t)pb.N};
            cuuint64_t strides[2] = {(cuuint64_t)Cp * es_b, (cuuint64_t)Cp * es_b * g.P};
            cuuint32_t box[3] = {(cuuint32_t)(bf16 ? 64 : 32), 64, 1};
            cuuint32_t es[3] = {1, 1, 1};
            if (g_encode_tiled(&dst_map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                               in_ws, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return cudaErrorInvalidValue;
        }
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t persist = std::min<int64_t>(g.n_tiles, (int64_t)sms * 3);
        const size_t smem = 1024 + 65536 + 64;
        static SmemOptIn attr_set[2];
        cudaError_t e = bf16 ? attr_set[1].ensure(repack_tma<true>, smem) : attr_set[0].ensure(repack_tma<false>, smem);
        if (e != cudaSuccess) return e;
        if (ev) cudaEventRecord(ev[0], st);
        const unsigned grid = (unsigned)(g.n_ker + persist);
        g.pdl_from = (int)std::max<int64_t>(0, (int64_t)grid - (int64_t)sms * 3);
        if (bf16)
            repack_tma<true><<<grid, 128, smem, st>>>(ker, (__nv_bfloat16*)ker_ws, src_map, dst_map, g);
        else
            repack_tma<false><<<grid, 128, smem, st>>>(ker, (float*)ker_ws, src_map, dst_map, g);
        if (ev) cudaEventRecord(ev[1], st);
        return cudaGetLastError();
    }
    const int64_t n_in = with_in ? (int64_t)g.ptiles * g.ctiles * pb.N : g.n_pre;   // fused: Ker + prologue
    const int64_t grid = g.n_ker + n_in;
    if (grid >= (1ll << 31)) return cudaErrorInvalidValue;
    {
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g.pdl_from = (int)std::max<int64_t>(0, grid - (int64_t)sms * 8);   // ~ the last resident wave
    }
    const size_t smem = std::max<size_t>(64 * 65 * sizeof(float),
                                         (g.krows > 1 ? (size_t)g.krows * g.C : (size_t)g.cc) * g.RS * sizeof(float));
    const int mode = g.n_pre > 0 || (fz.zero_ptr && !with_in) ? 2 : (fz.zero_ptr ? 1 : 0);
    auto kern = [&](auto bf) {
        constexpr bool B = decltype(bf)::value;
        return mode == 2 ? repack_all<B, 2> : mode == 1 ? repack_all<B, 1> : repack_all<B, 0>;
    };
    auto kfn16 = kern(std::true_type{});
    auto kfn32 = kern(std::false_type{});
    if (smem > 48 * 1024) {   // very large R*S: one channel per K1 CTA still needs > 48 KB
        cudaError_t e = bf16 ? cudaFuncSetAttribute(kfn16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(kfn32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (ev) cudaEventRecord(ev[0], st);
    if (bf16)
        kfn16<<<(unsigned)grid, 256, smem, st>>>(in, ker, (__nv_bfloat16*)in_ws, (__nv_bfloat16*)ker_ws, g);
    else
        kfn32<<<(unsigned)grid, 256, smem, st>>>(in, ker, (float*)in_ws, (float*)ker_ws, g);
    if (ev) cudaEventRecord(ev[1], st);
    return cudaGetLastError();
}


// ---- tiny-C tap expansion (explicit im2col in the layout transform) --------
// For layers with a handful of input channels (the C = 3 stems: Table 1 Y0,
// R1) the tensor kernel's TMA im2col rows are 32 B each and there are R*S of
// them per pixel: the layer is bound by TMA row throughput, not bytes.  The
// expansion writes, per OUTPUT pixel, all R*S*C taps as channels --
//   In'[n][h][w][(r*S + s)*C + c] = In[n][c][U*h + D*r - ph][U*w + D*s - pw]
// (zero outside the input, zero for channels >= R*S*C) and
//   Ker'[k][(r*S + s)*C + c]      = Ker[k][c][r][s]
// -- so that the main kernel runs the equivalent 1x1 convolution with
// C' = R*S*C over H x W (Eq. 1 regrouped: the same products, summed in the
// k-block order of the 1x1 problem).  One launch: blocks [0, ker_blocks)
// write Ker', the rest In' (8 channels = one 16-B bf16 / two 16-B tf32
// stores per thread).  Triggers the dependent launch at the end of each
// block, so the main kernel's large CTAs do not take SMs from it.
struct ExpandGeom {
    int N, K, C, H, W, R, S, U, D, ph, pw, Hin, Win;
    int RSC, Cp, groups;              // groups = Cp / 8 (16-B bf16 / 32-B tf32 store units)
    int ker_blocks, xblocks;          // Ker' blocks; In' blocks per output row
    int64_t ker_elems;
};

// Per-channel (r, s, c) decode of the expanded layout, shared by a block:
// input-plane offset of channel c and the tap's row / column shift.
struct TapEntry {
    int coff, dr, ds;                 // c*Hin*Win, D*r, D*s; coff < 0: padding channel (j >= R*S*C)
};

template <bool BF16>
__global__ void __launch_bounds__(256) expand_taps(const float* __restrict__ in, const float* __restrict__ ker,
                                                   typename Elem<BF16>::T* __restrict__ in_ws,
                                                   typename Elem<BF16>::T* __restrict__ ker_ws, const ExpandGeom g) {
    extern __shared__ TapEntry tab[];
    if ((int)blockIdx.x < g.ker_blocks) {
        for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < g.ker_elems; e += (int64_t)g.ker_blocks * 256) {
            const int64_t k = e / g.Cp;
            const int j = (int)(e - k * g.Cp);
            float v = 0.0f;
            if (j < g.RSC) {
                const int rs = j / g.C, c = j - rs * g.C;
                v = __ldg(ker + (k * g.C + c) * (g.R * g.S) + rs);
            }
            ker_ws[e] = Elem<BF16>::cvt(v);
        }
    } else {
        // block b >= ker_blocks: output row (b - ker_blocks) / xblocks = n*H + h,
        // its (pixel, channel-group) units [xb*256, xb*256 + 256)
        for (int j = threadIdx.x; j < g.Cp; j += 256) {
            TapEntry t{-1, 0, 0};
            if (j < g.RSC) {
                const int rs = j / g.C, c = j - rs * g.C, r = rs / g.S, sx = rs - (rs / g.S) * g.S;
                t = TapEntry{c * g.Hin * g.Win, g.D * r, g.D * sx};
            }
            tab[j] = t;
        }
        __syncthreads();
        const int b = (int)blockIdx.x - g.ker_blocks;
        const int row = b / g.xblocks, xb = b - row * g.xblocks;
        const int n = row / g.H, h = row - (row / g.H) * g.H;
        const int e = xb * 256 + (int)threadIdx.x;
        const int w = e / g.groups;
        if (w < g.W) {
            const int j0 = (e - w * g.groups) * 8;
            const int ih0 = g.U * h - g.ph, iw0 = g.U * w - g.pw;
            const float* src = in + (int64_t)n * g.C * g.Hin * g.Win;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const TapEntry t = tab[j0 + i];
                const int ih = ih0 + t.dr, iw = iw0 + t.ds;
                v[i] = (t.coff >= 0 && (unsigned)ih < (unsigned)g.Hin && (unsigned)iw < (unsigned)g.Win)
                           ? __ldg(src + t.coff + ih * g.Win + iw) : 0.0f;
            }
            typename Elem<BF16>::T* dst = in_ws + (((int64_t)row * g.W + w) * g.Cp + j0);
            if (BF16) {
                uint4 o;
                o.x = pack2_bf16(v[0], v[1]);
                o.y = pack2_bf16(v[2], v[3]);
                o.z = pack2_bf16(v[4], v[5]);
                o.w = pack2_bf16(v[6], v[7]);
                *reinterpret_cast<uint4*>(dst) = o;
            } else {
                float4* d4 = reinterpret_cast<float4*>(dst);
                d4[0] = make_float4(to_tf32_rna(v[0]), to_tf32_rna(v[1]), to_tf32_rna(v[2]), to_tf32_rna(v[3]));
                d4[1] = make_float4(to_tf32_rna(v[4]), to_tf32_rna(v[5]), to_tf32_rna(v[6]), to_tf32_rna(v[7]));
            }
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");
}

cudaError_t launch_expand(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker, void* in_ws,
                          void* ker_ws, cudaStream_t st, cudaEvent_t* ev) {
    ExpandGeom g;
    g.N = pb.N; g.K = pb.K; g.C = pb.C; g.H = pb.H; g.W = pb.W; g.R = pb.R; g.S = pb.S;
    g.U = pb.U; g.D = pb.D; g.ph = pb.ph; g.pw = pb.pw; g.Hin = (int)pb.Hin(); g.Win = (int)pb.Win();
    g.RSC = pb.R * pb.S * pb.C;
    g.Cp = Cp;
    if (Cp % 8 || Cp < g.RSC || (int64_t)pb.C * pb.Hin() * pb.Win() >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
    g.groups = Cp / 8;
    g.ker_elems = (int64_t)pb.K * Cp;
    g.ker_blocks = (int)std::min<int64_t>((g.ker_elems + 255) / 256, 256);
    g.xblocks = (int)(((int64_t)pb.W * g.groups + 255) / 256);
    const int64_t blocks = g.ker_blocks + (int64_t)pb.N * pb.H * g.xblocks;
    if (blocks >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
    const dim3 grid((unsigned)blocks);
    const size_t smem = (size_t)Cp * sizeof(TapEntry);
    if (ev) cudaEventRecord(ev[0], st);
    if (bf16)
        expand_taps<true><<<grid, 256, smem, st>>>(in, ker, (__nv_bfloat16*)in_ws, (__nv_bfloat16*)ker_ws, g);
    else
        expand_taps<false><<<grid, 256, smem, st>>>(in, ker, (float*)in_ws, (float*)ker_ws, g);
    if (ev) cudaEventRecord(ev[1], st);
    return cudaGetLastError();
}

// ---- FP32-accurate tensor path: exact bf16 splitting (CONV_PATH_FP32_TC) ----
// Every fp32 value x splits EXACTLY into three bf16 pieces, each the
// round-to-nearest-even bf16 of the remainder so far:
//   x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1) = x - x0 - x1
// (each subtraction is exact: a value and its nearest bf16 are within a
// factor 2; a binary32 significand is 24 bits, each piece takes 8 of them,
// so the third remainder fits a bf16 exactly).  x*y = sum_{i,j} x_i*y_j, and
// every x_i*y_j is exact in fp32 (8 x 8 significant bits).  The path computes
// the pairs (i, j) of split_pairs() -- i + j <= 2 (6 pairs; the three dropped
// are below 3 * 2^-24 |x*y|) or all 9 (exact products) -- as ONE bf16
// convolution with C' = npairs * Cq channels: In' channel p*Cq + c holds
// piece ip[p] of In channel c, Ker' channel p*Cq + c piece kp[p] of Ker
// channel c, so the tensor kernel's fp32 accumulation sums exactly those
// products (channels c >= C and the tail up to Cp are zero).
struct SplitGeom {
    int C, Cq, Cp, RS, npairs;
    int ip[kSplitMaxPairs], kp[kSplitMaxPairs];
    int K;
    int64_t P;                       // pixels per input image
    int ptiles, ctiles;              // K2 tile grid per image (64 px x 64 channels of In)
    int ker_blocks;
    int64_t ker_groups;              // K * RS * Cp / 8 (8 channels = one 16-B store)
    int* zero_ptr;                   // split-K arrival counters to clear
    int zero_n;
    int in_pairs;                    // In' piece blocks: npairs (pair layout) or 3 (compact: piece q at q*Cq)
    int in_cp;                       // In' channels per pixel
};

__device__ __forceinline__ void split3_bf16(float x, float (&v)[3]) {
    v[0] = __bfloat162float(__float2bfloat16_rn(x));
    const float r1 = __fsub_rn(x, v[0]);
    v[1] = __bfloat162float(__float2bfloat16_rn(r1));
    v[2] = __fsub_rn(r1, v[1]);               // exactly representable in bf16
}

__global__ void __launch_bounds__(256) split_repack(const float* __restrict__ in, const float* __restrict__ ker,
                                                    __nv_bfloat16* __restrict__ in_ws,
                                                    __nv_bfloat16* __restrict__ ker_ws, const SplitGeom g) {
    __shared__ float tile[64][65];
    const int tid = threadIdx.x;
    if ((int)blockIdx.x < g.ker_blocks) {
        // ---- Ker' [K][R][S][Cp]: one 8-channel group per thread ----
        for (int i = blockIdx.x * 256 + tid; i < g.zero_n; i += g.ker_blocks * 256) g.zero_ptr[i] = 0;
        const int gpr = g.Cp / 8;                  // groups per (k, rs) row
        for (int64_t e = (int64_t)blockIdx.x * 256 + tid; e < g.ker_groups; e += (int64_t)g.ker_blocks * 256) {
            const int64_t row = e / gpr;           // k * RS + rs
            const int j0 = (int)(e - row * gpr) * 8;
            const int64_t k = row / g.RS;
            const int rs = (int)(row - k * g.RS);
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int j = j0 + i, p = j / g.Cq, c = j - p * g.Cq;
                float x = 0.0f;
                if (p < g.npairs && c < g.C) {
                    float pc[3];
                    split3_bf16(__ldg(ker + (k * g.C + c) * g.RS + rs), pc);
                    const int kp = g.kp[p];
                    x = kp == 0 ? pc[0] : (kp == 1 ? pc[1] : pc[2]);
                }
                v[i] = x;
            }
            uint4 o;
            o.x = pack2_bf16(v[0], v[1]);
            o.y = pack2_bf16(v[2], v[3]);
            o.z = pack2_bf16(v[4], v[5]);
            o.w = pack2_bf16(v[6], v[7]);
            *reinterpret_cast<uint4*>(ker_ws + row * g.Cp + j0) = o;
        }
    } else {
        // ---- In' [N][Hin][Win][Cp]: one (image, 64-channel, 64-pixel) tile ----
        int b = (int)blockIdx.x - g.ker_blocks;
        const int pt = b % g.ptiles;
        b /= g.ptiles;
        const int ct = b % g.ctiles;
        const int64_t n = b / g.ctiles;
        const int64_t P = g.P, p0 = (int64_t)pt * 64;
        const int c0 = ct * 64;
        const float* src = in + n * g.C * P;
        if ((P & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = tid + i * 256;
                const int cl = idx >> 4, pq = (idx & 15) * 4;
                const int c = c0 + cl;
                const int64_t p = p0 + pq;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c < g.C && p < P) v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)c * P + p));
                tile[cl][pq] = v.x; tile[cl][pq + 1] = v.y; tile[cl][pq + 2] = v.z; tile[cl][pq + 3] = v.w;
            }
        } else {
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
                const int idx = tid + i * 256;
                const int cl = idx >> 6, pl = idx & 63;
                const int c = c0 + cl;
                const int64_t p = p0 + pl;
                tile[cl][pl] = (c < g.C && p < P) ? __ldg(src + (int64_t)c * P + p) : 0.0f;
            }
        }
        __syncthreads();
        __nv_bfloat16* dst = in_ws + n * P * g.in_cp;
#pragma unroll
        for (int i = 0; i < 2; ++i) {              // 64 px x 8 groups of 8 channels / 256 threads
            const int idx = tid + i * 256;
            const int pl = idx >> 3, cq = (idx & 7) * 8;
            const int64_t p = p0 + pl;
            const int c = c0 + cq;
            if (p < P && c < g.Cq) {
                float pc[8][3];
#pragma unroll
                for (int j = 0; j < 8; ++j) split3_bf16(tile[cq + j][pl], pc[j]);
                uint4 piece[3];
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    piece[q] = make_uint4(pack2_bf16(pc[0][q], pc[1][q]), pack2_bf16(pc[2][q], pc[3][q]),
                                          pack2_bf16(pc[4][q], pc[5][q]), pack2_bf16(pc[6][q], pc[7][q]));
                __nv_bfloat16* d = dst + p * g.in_cp + c;
                for (int pr = 0; pr < g.in_pairs; ++pr) {
                    const int q = g.in_pairs == 3 ? pr : g.ip[pr];
                    *reinterpret_cast<uint4*>(d + pr * g.Cq) = q == 0 ? piece[0] : (q == 1 ? piece[1] : piece[2]);
                }
            }
        }
        // the channel tail [npairs * Cq, Cp) is zero (written once, by the
        // first channel tile of each pixel block)
        const int tail0 = g.in_pairs * g.Cq, tail_groups = (g.in_cp - tail0) / 8;
        if (ct == 0 && tail_groups > 0) {
            for (int idx = tid; idx < 64 * tail_groups; idx += 256) {
                const int pl = idx / tail_groups, gq = idx - pl * tail_groups;
                const int64_t p = p0 + pl;
                if (p < P) *reinterpret_cast<uint4*>(dst + p * g.in_cp + tail0 + gq * 8) = make_uint4(0, 0, 0, 0);
            }
        }
    }
    // the main kernel waits for this grid's completion (griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;");
}

cudaError_t launch_split(const Problem& pb, int Cp, int npairs, const float* in, const float* ker, void* in_ws,
                         void* ker_ws, cudaStream_t st, cudaEvent_t* ev, int* zero_ptr, int zero_n, bool compact) {
    SplitGeom g;
    const SplitPairs sp = split_pairs(npairs);
    if (sp.n == 0) return cudaErrorInvalidValue;
    g.C = pb.C;
    g.Cq = split_cq(pb.C);
    g.Cp = Cp;
    g.RS = pb.R * pb.S;
    g.npairs = sp.n;
    for (int i = 0; i < kSplitMaxPairs; ++i) {
        g.ip[i] = sp.ip[i];
        g.kp[i] = sp.kp[i];
    }
    if (Cp % 8 || Cp < g.npairs * g.Cq) return cudaErrorInvalidValue;
    g.in_pairs = compact ? 3 : g.npairs;
    g.in_cp = compact ? 3 * g.Cq : Cp;
    g.K = pb.K;
    g.P = pb.Hin() * pb.Win();
    g.ptiles = (int)((g.P + 63) / 64);
    g.ctiles = (pb.C + 63) / 64;
    g.ker_groups = (int64_t)pb.K * g.RS * Cp / 8;
    g.ker_blocks = (int)std::min<int64_t>((g.ker_groups + 255) / 256, 1184);
    g.zero_ptr = zero_ptr;
    g.zero_n = zero_ptr ? zero_n : 0;
    const int64_t blocks = g.ker_blocks + (int64_t)g.ptiles * g.ctiles * pb.N;
    if (blocks >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
    if (ev) cudaEventRecord(ev[0], st);
    split_repack<<<(unsigned)blocks, 256, 0, st>>>(in, ker, (__nv_bfloat16*)in_ws, (__nv_bfloat16*)ker_ws, g);
    if (ev) cudaEventRecord(ev[1], st);
    return cudaGetLastError();
}

}  // namespace conv

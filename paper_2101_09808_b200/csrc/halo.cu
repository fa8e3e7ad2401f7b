// halo.cu -- K3h: single-launch tcgen05 convolution with shared-memory halo
// reuse, for small-C layers ("evaluate SMEM halo
// reuse").
//
// Eq. 1 over the PADDED output grid of an image: pixel index
// p = h * Win + w with w in [0, Win) (columns W..Win-1 are junk and never
// stored).  On that grid filter tap (r, s) reads input pixel p + r*Win + s,
// a pure shift, so the im2col operand of every tap is the same NHWC input
// tile viewed from row r*Win + s: the tile is staged in shared memory ONCE
// (tcgen05 descriptors may start at any row of a swizzled K-major tile --
// the swizzle follows absolute shared-memory address bits;
// scripts/probe_shift.cu measured every row shift 0..7 exact with base
// offset 0, SW64 and SW128) and the R*S taps are R*S descriptor offsets.
//
// Two launches, overlapped by programmatic dependent launch:
//   halo_ker_pack: Ker KCRS fp32 -> the B image, per-tap K-major swizzled
//      [BN rows][row bytes] tiles exactly as shared memory holds them (RNE
//      bf16 / RNA tf32; rows k >= K, channels >= C zero) -- converted once,
//      not once per CTA (a per-CTA conversion was measured 2x slower: its
//      strided L2 loads serialise on latency);
//   conv_halo_tcgen05, one CTA (8 warps) per 128-pixel tile of one image, all
//   K output channels (BN = K rounded up to 32..256):
//   1. thread 0: cp.async.bulk of the tile's input pixel range (plus halo,
//      (R-1)*Win + S-1 pixels) from every NCHW fp32 channel plane into an
//      fp32 staging area; warp 0 allocates TMEM;
//   2. all threads: staging -> the swizzled K-major A tile (one row per
//      input pixel, channels C..Cp-1 zero) -- all of this overlaps the pack;
//   3. thread 0, right after the input copies: griddepcontrol.wait, then
//      ONE bulk copy of the B image (its latency overlaps step 2);
//   4. thread 0: R*S*(row bytes / 32) tcgen05.mma (M = 128, N = BN) into TMEM,
//      tap (r, s) = A descriptor start + (r*Win + s) rows;
//   5. all warps: TMEM -> registers -> NCHW Out (valid pixels only).
// No NHWC workspace (only the small B image).  The k-order per output
// (tap-major, channels ascending within a tap) equals the im2col kernel's
// for one channel block, so results are bit-identical to it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace conv {

using namespace sm100;

struct HaloParams {
    const float* in;
    const float* ker;
    float* out;
    const uint8_t* bimg;   // the B image (halo_ker_pack output, R*S*b_tap_bytes)
    int N, K, C, H, W, R, S, Hin, Win;
    int Cp;            // channels per A/B row (16 / 32 / 64 bf16; 8 / 16 / 32 tf32): rowb = Cp * elem
    int rowb;          // bytes per operand row = swizzle span (32 / 64 / 128)
    int rows_a;        // A tile rows: 128 + (R-1)*Win + S-1, rounded up to 8
    int stage_px;      // fp32 staging pixels per channel: rows_a rounded up to 4 (16-B bulk copies)
    int tiles;         // 128-pixel tiles per image over the padded grid (H * Win pixels)
    int P;             // Hin * Win
    uint32_t a_off, b_off, st_off;   // smem offsets (1024-aligned)
    uint32_t b_tap_bytes;            // BN * rowb
};

__device__ __forceinline__ uint32_t halo_swz(int row, int chunk, int rowb) {
    // K-major SWIZZLE_{32,64,128}B: 16-B chunk index XOR row bits 7.. of the address
    const int x = rowb == 128 ? (row & 7) : rowb == 64 ? ((row >> 1) & 3) : ((row >> 2) & 1);
    return (uint32_t)(row * rowb + (((chunk ^ x) & (rowb / 16 - 1)) << 4));
}

__device__ __forceinline__ float halo_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t halo_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// 16 B of converted channels [c0, c0 + 8 / 4) of one row from 8 / 4 floats
template <bool BF16>
__device__ __forceinline__ uint4 halo_pack(const float* v) {
    if (BF16)
        return make_uint4(halo_bf16x2(v[0], v[1]), halo_bf16x2(v[2], v[3]), halo_bf16x2(v[4], v[5]),
                          halo_bf16x2(v[6], v[7]));
    return make_uint4(__float_as_uint(halo_tf32(v[0])), __float_as_uint(halo_tf32(v[1])),
                      __float_as_uint(halo_tf32(v[2])), __float_as_uint(halo_tf32(v[3])));
}

// Ker KCRS fp32 -> B image (per tap: BN rows of rowb bytes, K-major
// swizzled); one thread per 16-B chunk.  Triggers the dependent launch at
// once: the halo kernel's prologue (input staging) overlaps this grid.
template <bool BF16>
__global__ void __launch_bounds__(256) halo_ker_pack(const HaloParams p, uint8_t* __restrict__ bimg, int bn) {
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr int kEpc = BF16 ? 8 : 4;
    const int RS = p.R * p.S, nq = p.rowb / 16;
    const int64_t total = (int64_t)RS * bn * nq;
    for (int64_t e = blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
        const int q = (int)(e % nq);
        const int64_t row = e / nq;                     // tap * bn + k
        const int tap = (int)(row / bn), k = (int)(row - (int64_t)tap * bn);
        float v[8];
#pragma unroll
        for (int j = 0; j < kEpc; ++j) {
            const int c = q * kEpc + j;
            v[j] = (k < p.K && c < p.C) ? __ldg(p.ker + ((int64_t)k * p.C + c) * RS + tap) : 0.0f;
        }
        *reinterpret_cast<uint4*>(bimg + (size_t)tap * p.b_tap_bytes + halo_swz(k, q, p.rowb)) = halo_pack<BF16>(v);
    }
}

static constexpr int kThreadsH = 256;   // 8 warps: two per TMEM lane quadrant

template <int BN, bool BF16>
__global__ void __launch_bounds__(kThreadsH, 1) conv_halo_tcgen05(const HaloParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem + p.a_off;
    uint8_t* B = smem + p.b_off;
    float* stage = reinterpret_cast<float*>(smem + p.st_off);
    __shared__ __align__(8) uint64_t bar_in, bar_b, bar_mma;
    __shared__ uint32_t tmem_slot;
    constexpr int kEpc = BF16 ? 8 : 4;                 // elements per 16-B chunk
    constexpr uint32_t kCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n = blockIdx.x / p.tiles;
    const int p0 = (blockIdx.x - n * p.tiles) * 128;   // first padded-grid pixel of the tile
    const int npx = min(p.stage_px, p.P - p0);          // input pixels staged (multiple of 4: P % 4 == 0)

    // 1. bulk copies of the input pixel range, one per channel plane
    if (tid == 0) {
        mbar_init(&bar_in, 1);
        mbar_init(&bar_b, 1);
        mbar_init(&bar_mma, 1);
        fence_barrier_init();
        const uint32_t bytes = (uint32_t)npx * 4;
        mbar_arrive_expect_tx(&bar_in, bytes * (uint32_t)p.C);
        const float* src = p.in + ((int64_t)n * p.C) * p.P + p0;
        for (int c = 0; c < p.C; ++c)
            bulk_load_g2s(stage + (size_t)c * p.stage_px, src + (int64_t)c * p.P, bytes, &bar_in);
        // the B image, written by the pack grid (programmatic dependency):
        // requested now, so that its latency overlaps the input conversion
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint32_t bbytes = (uint32_t)(p.R * p.S) * p.b_tap_bytes;
        mbar_arrive_expect_tx(&bar_b, bbytes);
        for (uint32_t o = 0; o < bbytes; o += 32768)
            bulk_load_g2s(B + o, p.bimg + o, min(32768u, bbytes - o), &bar_b);
    }
    if (warp == 0) tmem_alloc(&tmem_slot, kCols);
    __syncthreads();                                    // barrier inits visible to every waiter

    const int chunks = p.rowb / 16;

    // 2. staged input -> A rows (pixel r of the tile's range), once landed;
    // a unit = 4 consecutive pixels x one 16-B channel chunk: kEpc LDS.128
    // (one per channel, 4 pixels each), 4 STS.128 (one per pixel row)
    mbar_wait(&bar_in, 0);
    {
        const int groups = p.rows_a / 4;               // rows_a is a multiple of 8
        for (int u = tid; u < groups * chunks; u += kThreadsH) {
            const int q = u / groups, r0 = (u - q * groups) * 4;
            float4 x[8];
#pragma unroll
            for (int e = 0; e < kEpc; ++e) {
                const int c = q * kEpc + e;
                x[e] = c < p.C ? *reinterpret_cast<const float4*>(stage + (size_t)c * p.stage_px + r0)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float v[8];
#pragma unroll
                for (int e = 0; e < kEpc; ++e) v[e] = i == 0 ? x[e].x : i == 1 ? x[e].y : i == 2 ? x[e].z : x[e].w;
                *reinterpret_cast<uint4*>(A + halo_swz(r0 + i, q, p.rowb)) = halo_pack<BF16>(v);
            }
        }
    }
    fence_proxy_async_smem();                           // generic smem writes -> tensor core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    // 4. the MMAs: tap (r, s) reads the A tile from row r*Win + s; the
    // whole warp runs the loop (descriptors in uniform registers), one
    // elected lane issues.  (Traced r02 on det: the 18 dependent N = 64 MMAs
    // into one accumulator take ~1.6 us -- ~180 cycles each, the MMA
    // latency, not its 50-cycle issue interval.)
    if (warp == 0) {
        mbar_wait(&bar_b, 0);
        const uint32_t layout = umma_layout_for_swizzle((uint32_t)p.rowb);
        const uint32_t idesc = make_idesc(BF16 ? 1u : 2u, 128, BN);
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
        const int ksteps = p.rowb / 32;
        uint32_t accum = 0;
        for (int r = 0; r < p.R; ++r)
            for (int s = 0; s < p.S; ++s) {
                const uint64_t ad = make_sdesc(a0 + (uint32_t)(r * p.Win + s) * p.rowb, 8 * p.rowb, layout);
                const uint64_t bd = make_sdesc(b0 + (uint32_t)(r * p.S + s) * p.b_tap_bytes, 8 * p.rowb, layout);
                if (elect_one_sync()) {
                    for (int kk = 0; kk < ksteps; ++kk) {
                        if (BF16) mma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, accum | (uint32_t)kk);
                        else mma_tf32(tmem, ad + 2 * kk, bd + 2 * kk, idesc, accum | (uint32_t)kk);
                    }
                }
                __syncwarp();
                accum = 1;
            }
        if (elect_one_sync()) tc_commit(&bar_mma);
        __syncwarp();
    }

    // 5. epilogue: warp w owns TMEM lanes 32(w%4).. = tile pixels
    // p0 + 32(w%4) + lane and the column half w/4 (32-column steps)
    mbar_wait_sleep(&bar_mma, 0, 64);
    tc_fence_after();
    const int qd = warp & 3;
    const int pix = p0 + qd * 32 + lane;
    const int h = pix / p.Win, w = pix - h * p.Win;
    const bool valid = h < p.H && w < p.W;
    float* obase = p.out + ((int64_t)n * p.K) * p.H * p.W + (int64_t)h * p.W + w;
    const int64_t HW = (int64_t)p.H * p.W;
#pragma unroll 1
    for (int j0 = (warp >> 2) * 32; j0 < BN; j0 += 64) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)j0, v);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j0 + j < p.K) __stcs(obase + (int64_t)(j0 + j) * HW, __uint_as_float(v[j]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, kCols);
    }
}

// ---- host -----------------------------------------------------------------

static bool halo_geometry(const Problem& pb, bool bf16, size_t smem_optin, HaloParams& p, int& bn, size_t& smem) {
    if (pb.U != 1 || pb.D != 1 || pb.ph != 0 || pb.pw != 0) return false;
    const int elem = bf16 ? 2 : 4;
    const int cbytes = pb.C * elem;
    const int rowb = cbytes <= 32 ? 32 : cbytes <= 64 ? 64 : cbytes <= 128 ? 128 : 0;
    if (!rowb || pb.K > 256) return false;
    const int64_t P = pb.Hin() * pb.Win();
    if (P % 4 || P >= (1ll << 30) || pb.Win() > 4096) return false;   // 16-B bulk copies of plane ranges
    bn = (pb.K + 15) / 16 * 16;
    if (bn < 32) bn = 32;
    bn = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;        // instantiated widths
    p.Cp = rowb / elem;
    p.rowb = rowb;
    const int64_t halo = (int64_t)(pb.R - 1) * pb.Win() + (pb.S - 1);
    p.rows_a = (int)((128 + halo + 7) / 8 * 8);
    p.stage_px = (p.rows_a + 3) / 4 * 4;
    const size_t a_bytes = (size_t)p.rows_a * rowb;
    p.b_tap_bytes = (uint32_t)((size_t)bn * rowb);
    const size_t b_bytes = (size_t)pb.R * pb.S * p.b_tap_bytes;
    const size_t st_bytes = (size_t)pb.C * p.stage_px * 4;
    auto up = [](size_t x) { return (x + 1023) / 1024 * 1024; };
    p.a_off = 0;
    p.b_off = (uint32_t)up(a_bytes);
    p.st_off = (uint32_t)(p.b_off + up(b_bytes));
    smem = 1024 + p.st_off + st_bytes;
    if (smem > smem_optin) return false;
    p.N = pb.N; p.K = pb.K; p.C = pb.C; p.H = pb.H; p.W = pb.W; p.R = pb.R; p.S = pb.S;
    p.Hin = (int)pb.Hin(); p.Win = (int)pb.Win();
    p.P = (int)P;
    p.tiles = (int)(((int64_t)pb.H * pb.Win() + 127) / 128);
    return (int64_t)pb.N * p.tiles < (1ll << 31);
}

bool halo_ok(const Problem& pb, bool bf16, size_t smem_optin) {
    HaloParams p;
    int bn;
    size_t smem;
    return halo_geometry(pb, bf16, smem_optin, p, bn, smem);
}

int64_t halo_ctas(const Problem& pb) { return (int64_t)pb.N * ((pb.H * pb.Win() + 127) / 128); }

template <int BN, bool BF16>
static cudaError_t launch_halo_t(const HaloParams& p, int grid, size_t smem, cudaStream_t st) {
    static SmemOptIn opt;
    auto kfn = conv_halo_tcgen05<BN, BF16>;
    if (cudaError_t e = opt.ensure(kfn, smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreadsH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlaps the pack grid
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, p);
}

size_t halo_ws_bytes(const Problem& pb, bool bf16) {
    const int elem = bf16 ? 2 : 4;
    const int cbytes = pb.C * elem;
    const int rowb = cbytes <= 32 ? 32 : cbytes <= 64 ? 64 : 128;
    int bn = (pb.K + 15) / 16 * 16;
    bn = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
    return (size_t)pb.R * pb.S * bn * rowb;
}

cudaError_t halo_run(const Problem& pb, bool bf16, const float* in, const float* ker, float* out, void* ws,
                     cudaStream_t st, cudaEvent_t* ev, std::string& err) {
    HaloParams p;
    int bn;
    size_t smem;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (!halo_geometry(pb, bf16, (size_t)optin, p, bn, smem)) { err = "layer not eligible for the halo kernel"; return cudaErrorInvalidValue; }
    p.in = in;
    p.ker = ker;
    p.out = out;
    p.bimg = static_cast<const uint8_t*>(ws);
    if (!ws) { err = "the halo kernel needs its B-image workspace"; return cudaErrorInvalidValue; }
    const int grid = (int)halo_ctas(pb);
    if (ev) cudaEventRecord(ev[0], st);
    const int64_t chunks = (int64_t)pb.R * pb.S * bn * (p.rowb / 16);
    const int pblocks = (int)std::min<int64_t>((chunks + 255) / 256, 592);
    if (bf16) halo_ker_pack<true><<<pblocks, 256, 0, st>>>(p, static_cast<uint8_t*>(ws), bn);
    else halo_ker_pack<false><<<pblocks, 256, 0, st>>>(p, static_cast<uint8_t*>(ws), bn);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = "halo Ker pack launch failed"; return e; }
    if (ev) cudaEventRecord(ev[1], st);
    switch (bn) {
        case 32: e = bf16 ? launch_halo_t<32, true>(p, grid, smem, st) : launch_halo_t<32, false>(p, grid, smem, st); break;
        case 64: e = bf16 ? launch_halo_t<64, true>(p, grid, smem, st) : launch_halo_t<64, false>(p, grid, smem, st); break;
        case 128: e = bf16 ? launch_halo_t<128, true>(p, grid, smem, st) : launch_halo_t<128, false>(p, grid, smem, st); break;
        default: e = bf16 ? launch_halo_t<256, true>(p, grid, smem, st) : launch_halo_t<256, false>(p, grid, smem, st); break;
    }
    if (e != cudaSuccess) { err = std::string("halo kernel launch failed: ") + cudaGetErrorString(e); return e; }
    if (ev) cudaEventRecord(ev[2], st);
    return cudaSuccess;
}

}  // namespace conv

// tc.cu -- K3: tcgen05 implicit-GEMM convolution.
//
// Eq. 1 as a GEMM: M = N*H*W output pixels, N_gemm = K output
// channels, K_gemm = R*S*C taps.  A[m, (r,s,c)] = In_NHWC[n, h+r, w+s, c] is
// loaded per (r, s, c-block) by TMA in im2col mode (the traversal walks BM
// consecutive output pixels, the filter-tap offsets (s, r) are added to every
// pixel); B[k, (r,s,c)] = Ker_KRSC[k, r, s, c] by a tiled TMA load.  Both
// operands are K-major with the 32/64/128-B swizzle matching the k-block's
// byte width.  tcgen05.mma (M = 128, N = BN) accumulates fp32 in TMEM.
//
// Warp roles (384 threads, one CTA per SM, persistent over tiles).  The
// warp arbiter favours higher warp ids, so the latency-critical issuers get
// the highest ones:
//   warp 11   MMA issuer (elected lane)   -> empty[stage] (tcgen05.commit)
//                                          -> tmem_full[acc]
//   warp 10   TMA producer (elected lane) -> full[stage]  (mbarrier, tx bytes)
//   warp 8    TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7 epilogue: tcgen05.ld 32x32b (warp w%4 owns TMEM lanes 32(w%4)..)
//             -> coalesced st.global into NCHW Out (consecutive TMEM lanes are
//             consecutive pixels of one (n,k) plane)   -> tmem_empty[acc]
//   warp 9    (fuse = 1) watcher: acquires the flags of the chunks each of
//             the CTA's (tile, channel block) units reads -> ready_ctr (smem)
//   warp 8    TMEM allocator; (fuse = 1) flag publisher: releases the flags
//             of the chunks this CTA's converters stored
//   warps 0-3 (fuse = 1) cooperative In transform: cp.async of NCHW fp32
//             chunks, RNE bf16 / RNA tf32 conversion, stores into the NHWC
//             workspace; then half of the CTA's last accumulator
// k-loop order: c-block outermost, then r, then s; a pipeline stage holds
// kbs consecutive iterations of that order.
//
// Accumulation order per output element is fixed by the k-loop (r, s, c-block
// ascending) and does not depend on the tile shape or on the grid, so results
// are bit-identical across BN choices and batch shards.
// Parallelism is over the non-reduction dims only (Sec. 7).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "internal.h"
#include "sm100.cuh"

namespace conv {

using namespace sm100;

static constexpr int kBM = 128;
static constexpr int kThreads = 384;
static constexpr int kRing = 64;            // fused transform: decoded-chunk ring entries
static constexpr int kDecode = 16;          //   decoded per block, one block ahead
static constexpr int kMaxTnb = 6;           //   chunk buffers at most
// The CTA's last tile is stored by 8 warps (4-7 and 0-3) when BN allows two
// 32-column halves (CONV_DEBUG_MODE bit 32 disables it, experiments only).
#ifndef CONV_ENABLE_TRACE
#define CONV_ENABLE_TRACE 0   // build with CONV_BUILD_TRACE=1 (build.py) for scripts/trace_tc.py
#endif
static constexpr bool kTraceBuild = CONV_ENABLE_TRACE != 0;

#ifndef CONV_SPLIT_LAST
#define CONV_SPLIT_LAST 1
#endif        // 12 warps: 4 In-transform, 4 epilogue, alloc, watcher, TMA, MMA

struct TcParams {
    float* out;
    int M;            // N*H*W
    int HW;           // H*W
    int W;            // output width
    int K;            // output channels
    int R, S;
    int U;            // stride: the im2col traversal visits input pixels U apart
    int D;            // dilation: tap (r, s) is the im2col offset (D*s, D*r)
    int ph, pw;       // zero padding: output (h, w)'s window starts at input (U*h - ph, U*w - pw)
    int Cp, bkc, n_cblk;
    int k_iters;      // R*S*n_cblk
    int num_n_tiles;
    int num_tiles;
    // split-K (fuse = 0, one wave): work item w = (tile w / splits, split
    // w % splits) covers k iterations [split * kper, min(k_iters, (split + 1)
    // * kper)) of the fixed k order; each writes an fp32 partial slab, waits
    // for the tile's other splits, then sums a 1/splits column share of the
    // slabs in split order into Out
    int splits;
    int kper;                 // k iterations per split (a multiple of kbs)
    int num_work;             // num_tiles * splits
    float* part;              // [num_work][CG][BN][128] partial slabs
    int* tile_ctr;            // [num_tiles][CG] arrivals (zeroed by the repack launch)
    int stages;
    int kbs;                  // k-blocks per pipeline stage (1, 2 or 4)
    uint32_t sw;              // 32 / 64 / 128 (bytes per operand row per k-block)
    uint32_t a_stage_bytes;   // kbs * 128 * sw
    uint32_t b_stage_bytes;   // kbs * (bn / cg) * sw
    unsigned long long* trace;  // experiments only (env CONV_TRACE): per-CTA timeline, 64 slots
    // ---- cooperative In transform (a-3 inside the main kernel, fuse = 1) ----
    int fuse;                 // 1: warps 0-3 of every CTA convert NCHW fp32 chunks into the NHWC workspace
    int* flags;               // [Q][nch] chunk-ready flags (zeroed by the Ker repack launch)
    const float* in;          // In, NCHW fp32
    void* in_ws;              // NHWC workspace
    int C;                    // input channels
    int P, Win, Hin;          // pixels per input image (Hin*Win), input width, height
    int npch;                 // 64-pixel chunks per image plane: ceil(P / 64)
    int cc;                   // channels per chunk (min(32, bkc))
    int nch;                  // channel chunks: Cp / cc
    int hh;                   // channel chunks per k-block: bkc / cc
    int total_chunks;         // N * npch * nch
    int seq0;                 // sequence indices [0, seq0) were converted by the repack launch (prologue)
    int hh_log2;              // log2(hh)
    int n_groups;             // chunk groups (waves of the schedule, merged to <= 32)
    int gend[32];             // group g covers chunk-pixel indices q in [gend[g-1], gend[g])
    int tnb;                  // input staging buffers (2..4)
    uint32_t tr_off;          // byte offset of the transform smem region (1024-aligned)
    // ---- promoted accumulation (FP32_TC plans, PROMOTE instances) ----
    int pnb;                  // compact FP32_TC In' (PROMOTE only): k-blocks per piece block (0: off);
    int pip[kSplitMaxPairs];  //   pair block p of the k loop reads In' piece pip[p]
    int pchunk;               // pipeline stages per promotion chunk: the tensor core accumulates a
                              // chunk of the k loop in TMEM (fresh accumulator), the epilogue warps add
                              // it to fp32 registers (IEEE round-to-nearest) -- the tcgen05 fp32
                              // accumulation alone truncates (reading R16)
};

// ---- cooperative NCHW -> NHWC transform (row a-3 inside K3) ----------------
// The input is cut into chunks (image n, 64-pixel run pch of the NCHW plane,
// cc channels), ordered by when the persistent schedule first needs them:
// waves of tiles, then channel block, then pixel.  CTA w of W transforms
// sequence entries w, w + W, ... (all CTAs are co-resident: one per SM, grid
// <= SM count).  A chunk is TMA-loaded as [cc][64] fp32,
// converted (RNA tf32 / RNE bf16) and transposed in place into a [64 px][cc]
// row-swizzled tile, TMA-stored into the NHWC workspace and published with
// a release flag.  Each CTA's watcher acquires the flags of the chunks its
// next (tile, channel block) im2col loads read and hands them to the TMA
// producer through a shared counter.
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta_smem(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_smem(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int4 lds_int4(const int4* p) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Chunk j of the sequence -> {flag index q*nch + ch, image n, first pixel,
// first channel}.  Group g = the q range [gend[g-1], gend[g]) first read by
// wave g of the persistent schedule (host-computed, see tc_run), so group g
// starts at sequence index gend[g-1]*nch; inside a group the order is
// (channel block, q, channel chunk within the block).
__device__ __forceinline__ int4 chunk_decode(const TcParams& p, int j) {
    int g = 0;
    while (g < p.n_groups - 1 && p.gend[g] * p.nch <= j) ++g;
    const int e_prev = g > 0 ? p.gend[g - 1] : 0;
    const int l = j - e_prev * p.nch;
    const int per_cb = (p.gend[g] - e_prev) << p.hh_log2;
    const int cb = l / per_cb;
    const int rem = l - cb * per_cb;
    const int q = e_prev + (rem >> p.hh_log2);
    const int ch = (cb << p.hh_log2) + (rem & ((1 << p.hh_log2) - 1));
    const int n = q / p.npch;
    return make_int4(q * p.nch + ch, n, (q - n * p.npch) * 64, ch * p.cc);
}

// Thread t of the 128 converters: pixel t & 63 of the chunk, channel half
// t >> 6 (cc/2 channels).  Reads its values from the [cc][64] fp32 smem
// copy of the chunk (conflict-free: consecutive lanes, consecutive pixels).
__device__ __forceinline__ void chunk_read(const float* tin, int cc, int tid, float (&v)[16]) {
    const int px = tid & 63, half = tid >> 6, ch = cc / 2;
    const float* s = tin + (half * ch) * 64 + px;
#pragma unroll
    for (int j = 0; j < 16; ++j)
        if (j < ch) v[j] = s[j * 64];
}
// In place: [cc][64] fp32 -> [64 px][cc] rows of cc*elem bytes, 16-B
// pieces swizzled as the destination map's SWIZZLE_{32,64,128}B expects
// (piece k of row r at k ^ ((r * row_bytes >> 7) & (row_bytes/16 - 1))).
// All threads read (chunk_read) before any thread writes.
template <bool BF16>
__device__ __forceinline__ void chunk_write(uint8_t* tout, int cc, int tid, const float (&v)[16]) {
    const int px = tid & 63, half = tid >> 6, ch = cc / 2;
    const int row_bytes = cc * (BF16 ? 2 : 4);
    const int sw = ((px * row_bytes) >> 7) & (row_bytes / 16 - 1);
    uint8_t* row = tout + px * row_bytes;
    if (BF16) {   // ch in {8, 16}: 8 channels per 16-B piece
        const int nk = ch / 8;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            if (kk < nk) {
                uint4 o;
                o.x = pack_bf16x2(v[8 * kk + 0], v[8 * kk + 1]);
                o.y = pack_bf16x2(v[8 * kk + 2], v[8 * kk + 3]);
                o.z = pack_bf16x2(v[8 * kk + 4], v[8 * kk + 5]);
                o.w = pack_bf16x2(v[8 * kk + 6], v[8 * kk + 7]);
                const int k = half * nk + kk;
                *reinterpret_cast<uint4*>(row + ((k ^ sw) << 4)) = o;
            }
        }
    } else {      // ch in {4, 8, 16}: 4 channels per 16-B piece
        const int nk = ch / 4;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            if (kk < nk) {
                float4 o;
                o.x = tf32_rna(v[4 * kk + 0]);
                o.y = tf32_rna(v[4 * kk + 1]);
                o.z = tf32_rna(v[4 * kk + 2]);
                o.w = tf32_rna(v[4 * kk + 3]);
                const int k = half * nk + kk;
                *reinterpret_cast<float4*>(row + ((k ^ sw) << 4)) = o;
            }
        }
    }
}

// TMEM accumulator columns [j_lo, j_hi) of one tile -> NCHW Out.  Warp
// quadrant q owns TMEM lanes 32q..32q+31 = the tile's pixels 32q + lane;
// each 32x32b load gives a thread 32 consecutive output channels of its
// pixel, stored as 32 coalesced 128-B runs (one per channel) by the warp.
template <int BN, int CG>
__device__ __forceinline__ void store_accumulator(const TcParams& p, uint32_t tmem_base, int tile, int acc,
                                                  uint32_t rank, int q, uint32_t lane, int j_lo, int j_hi) {
    const int m_tile = tile / p.num_n_tiles;
    const int n_tile = tile - m_tile * p.num_n_tiles;
    const int m = m_tile * (kBM * CG) + (int)rank * kBM + q * 32 + (int)lane;
    const int k0 = n_tile * BN;
    const bool valid_m = m < p.M;
    const int img = valid_m ? m / p.HW : 0;
    const int pix = valid_m ? m - img * p.HW : 0;
    float* obase = p.out + ((int64_t)img * p.K) * p.HW + pix;
    const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
    for (int j0 = j_lo; j0 < j_hi; j0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t0 + (uint32_t)j0, v);
        tmem_ld_wait();
        const int kbase = k0 + j0;
        if (valid_m) {
            if (kbase + 32 <= p.K) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    __stcs(obase + (int64_t)(kbase + j) * p.HW, __uint_as_float(v[j]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (kbase + j < p.K) __stcs(obase + (int64_t)(kbase + j) * p.HW, __uint_as_float(v[j]));
            }
        }
    }
}

// Split-K: this thread's accumulator row (TMEM lane q*32 + lane) of work
// item w -> its partial slab, column-major (a warp writes 128 contiguous B
// per column).
template <int BN, int CG>
__device__ __forceinline__ void store_partial(const TcParams& p, uint32_t tmem_base, int w, int acc, uint32_t rank,
                                              int q, uint32_t lane) {
    float* slab = p.part + ((size_t)w * CG + rank) * (kBM * BN) + q * 32 + lane;
    const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
    for (int j0 = 0; j0 < BN; j0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t0 + (uint32_t)j0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) __stcg(slab + (size_t)(j0 + j) * kBM, __uint_as_float(v[j]));
    }
}

// Split-K reduction share of split `sp` (CG = 1): columns [c_lo, c_hi) of
// the tile, staged in shared memory as `splits` consecutive [ncols][128]
// blocks (one per slab, bulk-copied from L2); this thread's row of each
// column is the sum of the slabs in split order 0, 1, ..., splits-1 (fixed,
// so the result is deterministic).
template <int BN>
__device__ __forceinline__ void reduce_share(const TcParams& p, int tile, const float* red, int c_lo, int c_hi,
                                             int q, uint32_t lane) {
    const int m_tile = tile / p.num_n_tiles;
    const int n_tile = tile - m_tile * p.num_n_tiles;
    const int row = q * 32 + (int)lane;
    const int m = m_tile * kBM + row;
    if (m >= p.M) return;
    const int k0 = n_tile * BN;
    const int img = m / p.HW, pix = m - img * p.HW;
    float* obase = p.out + ((int64_t)img * p.K + k0) * p.HW + pix;
    const int ncols = c_hi - c_lo, cend = min(c_hi, p.K - k0);
    const float* r = red + row;
#pragma unroll 1
    for (int c = c_lo; c < cend; ++c) {
        const float* rc = r + (c - c_lo) * kBM;
        float acc = rc[0];
#pragma unroll 4
        for (int sp = 1; sp < p.splits; ++sp) acc += rc[(size_t)sp * ncols * kBM];
        __stcs(obase + (int64_t)c * p.HW, acc);
    }
}

// CG = 1: one CTA per 128-pixel tile (tcgen05 cta_group::1, M = 128).
// CG = 2: a CTA pair (cluster of 2 on one TPC) per 256-pixel tile
//   (cta_group::2, M = 256): each CTA loads its own 128 A rows and HALF of
//   the BN B rows; the leader CTA issues the MMAs, which read both CTAs'
//   shared memory, and each CTA's TMEM receives its own 128 accumulator rows.
//   Per SM this halves the B operand traffic (L2 -> SMEM and SMEM -> tensor
//   core), which is what bounds the 1-CTA kernel on wide tiles.
template <int BN, bool BF16, int CG, int KSTEPS, bool SPLIT, bool FUSE, bool PROMOTE>
__global__ void __launch_bounds__(kThreads, 1)
conv_igemm_tcgen05(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b,
                   const __grid_constant__ CUtensorMap tmap_src,    // fuse: In NCHW fp32 {P, C, N}
                   const __grid_constant__ CUtensorMap tmap_dst,    // fuse: workspace NHWC {Cp, P, N}
                   const TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // timeline instrumentation (scripts/trace_tc.py) only in trace builds:
    // in production builds it folds away (its clock reads and branches sat
    // on the producer / MMA hot loops)
    unsigned long long* const trace = kTraceBuild ? p.trace : nullptr;
    // 1024-B alignment for the 128-B swizzle atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + (size_t)p.stages * p.a_stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_b + (size_t)p.stages * p.b_stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + p.stages;
    uint64_t* tmem_full = bars + 2 * p.stages;
    uint64_t* tmem_empty = tmem_full + 2;
    int* ready_ctr = reinterpret_cast<int*>(tmem_empty + 2);     // fuse: (tile, cb) units confirmed
    uint64_t* last_full = tmem_empty + 3;                        // the CTA's last accumulator is ready
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 4);
    int* done_ctr = reinterpret_cast<int*>(tmem_empty + 5);      // fuse: chunks stored so far
    int* pub_ctr = done_ctr + 1;                                 // fuse: chunks whose flags are published
    // fuse: per chunk buffer a "loaded" (TMA tx) and a "converted" (4 warps)
    // mbarrier, then the decoded-chunk counter, after the pipeline barriers
    uint64_t* tfull = tmem_empty + 6;
    uint64_t* tconv = tfull + kMaxTnb;
    int* dec_ctr = reinterpret_cast<int*>(tconv + kMaxTnb);      // fuse: ring entries decoded so far
    // transform region (fuse): tnb chunk buffers of [cc][64] fp32 and a
    // kRing-entry ring of decoded chunks
    uint8_t* tbuf = smem + p.tr_off;
    int4* cring = reinterpret_cast<int4*>(tbuf + (size_t)p.tnb * p.cc * 256);
    // static chunk assignment: CTA w of W takes sequence indices seq0 + w, seq0 + w + W, ...
    const int n_my = FUSE ? max(0, (p.total_chunks - p.seq0 - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) : 0;

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;       // position in the pair
    const bool leader = rank == 0;
    const int unit = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;   // pair / CTA index
    const int nunits = CG == 2 ? (int)nclusters_x() : (int)gridDim.x;

    if (threadIdx.x == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        if (FUSE) {
            prefetch_tmap(&tmap_src);
            prefetch_tmap(&tmap_dst);
            for (int i = 0; i < p.tnb; ++i) {
                mbar_init(&tfull[i], 1);
                mbar_init(&tconv[i], 4);                          // one arrive per converter warp
            }
            *done_ctr = 0;
            *pub_ctr = 0;
            *dec_ctr = 0;
        }
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            // one arrive per epilogue warp of the pair (8 warps promote)
            mbar_init(&tmem_empty[i], (PROMOTE ? 8 : 4) * CG);
        }
        mbar_init(last_full, 1);
        *ready_ctr = 0;
        fence_barrier_init();
    }
    if (warp == 8) {
        if (CG == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
        else tmem_alloc(tmem_slot, kTmemCols);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const bool kSplitLast = !SPLIT && !PROMOTE && CONV_SPLIT_LAST && BN >= 64;
    // Programmatic dependent launch: everything above overlapped the tail of
    // the repack launch; from here on the repacked workspace (and, fused, the
    // zeroed chunk flags) is read and Out written, so wait for the preceding
    // grid to complete and flush.
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 10) {
        // ===== TMA producer (both CTAs of a pair): the whole warp runs the
        // loop (warp-uniform control flow keeps the operands in uniform
        // registers), one elected lane issues =====
        {
            const uint64_t pol_a = policy_evict_normal();
            const uint64_t pol_b = policy_evict_last();   // Ker is re-read by every M tile
            const uint32_t tx_bytes = CG * (p.a_stage_bytes + p.b_stage_bytes);
            long long prod_wait = 0;
            int stage = 0;
            uint32_t phase = 0;
            int tiles_done = 0;                           // fuse: tiles of this CTA so far
            int ready_seen = 0;                           // fuse: last value read from ready_ctr
            long long ready_wait = 0;
            for (int wi = unit; wi < p.num_work; wi += nunits, ++tiles_done) {
                const int tile = SPLIT ? wi / p.splits : wi;
                const int it_beg = SPLIT ? (wi - tile * p.splits) * p.kper : 0;
                const int it_end = SPLIT ? min(p.k_iters, it_beg + p.kper) : p.k_iters;
                const int m_tile = tile / p.num_n_tiles;
                const int n_tile = tile - m_tile * p.num_n_tiles;
                const int m0 = m_tile * (kBM * CG) + (int)rank * kBM;
                const int img = m0 / p.HW;
                const int pix = m0 - img * p.HW;
                const int h0 = pix / p.W;
                const int w0 = pix - h0 * p.W;
                const int kb0 = n_tile * BN + (int)rank * (BN / CG);   // this CTA's B rows
                const uint32_t a_blk = kBM * p.sw, b_blk = (BN / CG) * p.sw;
                // k iterations in one fixed order -- (cb, r, s), s fastest --
                // tracked by counters (no divisions); a stage holds kbs
                // consecutive iterations, so the order does not depend on kbs
                // (results bit-identical across tilings, P10).
                int cb = 0, r = 0, s = 0;
                if (SPLIT && it_beg) {                    // split-K: start mid-order
                    s = it_beg % p.S;
                    r = (it_beg / p.S) % p.R;
                    cb = it_beg / (p.S * p.R);
                }
                for (int it0 = it_beg; it0 < it_end; it0 += p.kbs) {
                    const int cb_s = cb, r_s = r, s_s = s;
                    // advance the counters past this stage (all lanes, uniform)
                    int cb_last = cb;
                    for (int kb = 0; kb < p.kbs; ++kb) {
                        cb_last = cb;
                        if (++s == p.S) { s = 0; if (++r == p.R) { r = 0; ++cb; } }
                    }
                    if (FUSE) {
                        // the watcher has confirmed (tile, channel block) units in
                        // order; this stage reads channel blocks up to cb_last
                        const int need = tiles_done * p.n_cblk + cb_last + 1;
                        if (ready_seen < need) {
                            const long long t0 = clock64();
                            while ((ready_seen = ld_acquire_cta_smem(ready_ctr)) < need) {
                                __nanosleep(128);         // do not steal issue slots from the converters
                                if (clock64() - t0 > 8000000000ll) __trap();
                            }
                            fence_proxy_async_global();   // flags observed -> TMA reads of the workspace
                            if (trace) ready_wait += clock64() - t0;
                        }
                    }
                    const long long pw0 = trace ? clock64() : 0;
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (trace) prod_wait += clock64() - pw0;
                    uint8_t* a_dst = smem_a + (size_t)stage * p.a_stage_bytes;
                    uint8_t* b_dst = smem_b + (size_t)stage * p.b_stage_bytes;
                    if (elect_one_sync()) {
                        {
                            if (leader) mbar_arrive_expect_tx(&full[stage], tx_bytes);
                            int c1 = cb_s, r1 = r_s, s1 = s_s;
                            for (int kb = 0; kb < p.kbs; ++kb) {
                                const int bx = (r1 * p.S + s1) * p.Cp + c1 * p.bkc;
                                // compact FP32_TC In': pair block -> its piece's channels
                                int ca = c1 * p.bkc;
                                if constexpr (PROMOTE) {
                                    if (p.pnb) {
                                        const int pb_ = c1 / p.pnb;
                                        ca = (p.pip[pb_] * p.pnb + (c1 - pb_ * p.pnb)) * p.bkc;
                                    }
                                }
                                if (CG == 2) {
                                    tma_load_im2col_4d_pair(a_dst + kb * a_blk, &tmap_a, &full[stage], ca,
                                                            w0 * p.U - p.pw, h0 * p.U - p.ph, img, (uint16_t)(s1 * p.D), (uint16_t)(r1 * p.D), pol_a);
                                    tma_load_2d_pair(b_dst + kb * b_blk, &tmap_b, &full[stage], bx, kb0, pol_b);
                                } else {
                                    tma_load_im2col_4d(a_dst + kb * a_blk, &tmap_a, &full[stage], ca,
                                                       w0 * p.U - p.pw, h0 * p.U - p.ph, img, (uint16_t)(s1 * p.D), (uint16_t)(r1 * p.D), pol_a);
                                    tma_load_2d(b_dst + kb * b_blk, &tmap_b, &full[stage], bx, kb0, pol_b);
                                }
                                if (++s1 == p.S) { s1 = 0; if (++r1 == p.R) { r1 = 0; ++c1; } }
                            }
                        }
                    }
                    __syncwarp();
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                }
            }
            if (trace && lane == 0) {
                trace[(size_t)blockIdx.x * 64 + 60] = (unsigned long long)prod_wait;
                trace[(size_t)blockIdx.x * 64 + 61] = globaltimer_ns();
                trace[(size_t)blockIdx.x * 64 + 57] = (unsigned long long)ready_wait;
            }
        }
    } else if (warp == 11) {
        // ===== MMA issuer (leader CTA only): whole warp loops, one elected
        // lane issues the tcgen05 instructions =====
        if (leader) {
            constexpr uint32_t idesc = make_idesc(BF16 ? 1u : 2u, kBM * CG, BN);
            constexpr uint32_t kSw = KSTEPS * 32;            // swizzle span = k-block row bytes
            constexpr uint32_t layout = umma_layout_for_swizzle(kSw);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            // Descriptors: the stage-0 descriptor plus (byte offset >> 4) in
            // the start-address field; one k step of 32 B adds 2.
            const uint64_t a_desc0 = make_sdesc(smem_u32(smem_a), 8 * kSw, layout);
            const uint64_t b_desc0 = make_sdesc(smem_u32(smem_b), 8 * kSw, layout);
            const uint32_t a_step = p.a_stage_bytes >> 4, b_step = p.b_stage_bytes >> 4;
            constexpr uint32_t a_blk = (kBM * kSw) >> 4, b_blk = ((BN / CG) * kSw) >> 4;
            const int kbs = p.kbs;

            unsigned long long* tr = trace ? trace + (size_t)blockIdx.x * 64 : nullptr;
            int ti = 0;
            if (tr && lane == 0) tr[0] = globaltimer_ns();
            for (int wi = unit; wi < p.num_work; wi += nunits, ++ti) {
                const int tile = SPLIT ? wi / p.splits : wi;
                const int it_beg = SPLIT ? (wi - tile * p.splits) * p.kper : 0;
                const int iters = SPLIT ? (min(p.k_iters, it_beg + p.kper) - it_beg) / kbs : p.k_iters / kbs;
                // PROMOTE: the tile's k loop in chunks of pchunk stages, each
                // into a fresh (double-buffered) accumulator the epilogue adds
                // to its fp32 registers; otherwise one chunk = the whole loop
                const int chunk = PROMOTE ? p.pchunk : iters;
                for (int c0 = 0; c0 < iters; c0 += chunk) {
                const int c1 = min(iters, c0 + chunk);
                mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                if (tr && lane == 0 && ti < 8) tr[1 + 4 * ti] = globaltimer_ns();
                long long wait_cyc = 0;
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                uint32_t accum = 0;                      // first MMA of the tile (chunk) overwrites D
                for (int it = c0; it < c1; ++it) {
                    const long long w0 = tr ? clock64() : 0;
                    mbar_wait(&full[stage], phase);
                    if (tr) wait_cyc += clock64() - w0;
                    tc_fence_after();
                    if (elect_one_sync()) {
                        const uint64_t ad0 = a_desc0 + (uint64_t)(stage * a_step);
                        const uint64_t bd0 = b_desc0 + (uint64_t)(stage * b_step);
                        {
                            for (int kb = 0; kb < kbs; ++kb) {
#pragma unroll
                                for (int kk = 0; kk < KSTEPS; ++kk) {
                                    const uint64_t ad = ad0 + (uint64_t)(kb * a_blk + 2 * kk);
                                    const uint64_t bd = bd0 + (uint64_t)(kb * b_blk + 2 * kk);
                                    if (CG == 2) {
                                        if (BF16) mma_bf16_pair(d_tmem, ad, bd, idesc, accum);
                                        else      mma_tf32_pair(d_tmem, ad, bd, idesc, accum);
                                    } else {
                                        if (BF16) mma_bf16(d_tmem, ad, bd, idesc, accum);
                                        else      mma_tf32(d_tmem, ad, bd, idesc, accum);
                                    }
                                    accum = 1;
                                }
                            }
                        }
                        // frees the smem slot (in both CTAs) when the MMAs retire
                        if (CG == 2) tc_commit_pair_mc(&empty[stage], 0x3);
                        else tc_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                }
                // accumulator ready for the epilogue (of both CTAs); the last
                // tile's also signals warps 0-3, which store half of it
                if (elect_one_sync()) {
                    if (CG == 2) tc_commit_pair_mc(&tmem_full[acc], 0x3);
                    else tc_commit(&tmem_full[acc]);
                    if (kSplitLast && wi + nunits >= p.num_work) {
                        if (CG == 2) tc_commit_pair_mc(last_full, 0x3);
                        else tc_commit(last_full);
                    }
                }
                __syncwarp();
                if (tr && lane == 0 && ti < 8) {
                    tr[1 + 4 * ti + 1] = (unsigned long long)wait_cyc;
                    tr[1 + 4 * ti + 2] = globaltimer_ns();
                    tr[1 + 4 * ti + 3] = (unsigned long long)clock64();
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }   // chunks
            }
        }
    } else if (warp == 9) {
        // ===== watcher + publisher (fuse).  Each pass: (1) release the flags
        // of chunks whose stores the storer reports landed (done_ctr), up to
        // 32 per warp instruction, one GPU-scope fence per batch; (2) check
        // the next (tile, channel block) unit of this CTA -- relaxed reads of
        // the flags of every chunk its im2col loads read -- and, once all are
        // set, acquire them and hand the unit count to the TMA producer. =====
        if (FUSE) {
            int u = 0, pub = 0;
            const int n_units = ((p.num_tiles - unit + nunits - 1) / nunits) * p.n_cblk;
            int tile = unit, cb = 0, q_lo = 0, cnt = 0;
            auto tile_range = [&]() {
                const int m_tile = tile / p.num_n_tiles;
                const int m0 = m_tile * (kBM * CG) + (int)rank * kBM;
                q_lo = 0;
                int q_hi = -1;                            // empty if the rows are all past M
                if (m0 < p.M) {
                    const int m1 = min(m0 + kBM, p.M) - 1;
                    const int na = m0 / p.HW, nb = m1 / p.HW;
                    const int ha = (m0 - na * p.HW) / p.W, hb = (m1 - nb * p.HW) / p.W;
                    // input rows the tile's windows touch (padding rows clamped away)
                    const int ra = min(max(ha * p.U - p.ph, 0), p.Hin - 1);
                    const int rb = min(max(hb * p.U - p.ph + p.D * (p.R - 1), 0), p.Hin - 1);
                    q_lo = na * p.npch + (ra * p.Win) / 64;
                    q_hi = nb * p.npch + (rb * p.Win + p.Win - 1) / 64;
                }
                cnt = (q_hi - q_lo + 1) * p.hh;
            };
            if (n_units > 0) tile_range();
            long long w_spin = 0;
            long long t_last = clock64();                 // watchdog: time of the last progress
            while (u < n_units || pub < n_my) {
                bool progress = false;
                const int done = ld_acquire_cta_smem(done_ctr);
                if (pub < done) {
                    const int batch = min(32, done - pub);
                    if ((int)lane < batch) st_release_gpu(p.flags + cring[(pub + (int)lane) & (kRing - 1)].x, 1);
                    if (trace && lane == 0 && pub == 0) trace[(size_t)(512 + blockIdx.x) * 64 + 2] = globaltimer_ns();
                    pub += batch;
                    __syncwarp();
                    if (lane == 0) st_release_cta_smem(pub_ctr, pub);
                    progress = true;
                }
                if (u < n_units) {
                    bool ok = true;
                    for (int i = (int)lane; i < cnt; i += 32) {
                        const int q = q_lo + i / p.hh;
                        const int ch = cb * p.hh + (i - (i / p.hh) * p.hh);
                        if (ld_relaxed_gpu(p.flags + (size_t)q * p.nch + ch) == 0) ok = false;
                    }
                    if (__all_sync(0xffffffffu, ok)) {
                        fence_acq_rel_gpu();              // the flags read above -> acquire
                        fence_proxy_async_global();       // -> the producer's TMA reads
                        ++u;
                        if (lane == 0) st_release_cta_smem(ready_ctr, u);
                        if (trace && lane == 0 && u == 1) trace[(size_t)blockIdx.x * 64 + 56] = globaltimer_ns();
                        if (++cb == p.n_cblk) {
                            cb = 0;
                            tile += nunits;
                            if (u < n_units) tile_range();
                        }
                        progress = true;
                    }
                }
                if (!progress) {
                    const long long t0 = clock64();
                    __nanosleep(128);
                    if (trace) w_spin += clock64() - t0;
                    if (t0 - t_last > 8000000000ll) __trap();   // ~4 s without progress
                } else {
                    t_last = clock64();
                }
            }
            if (trace && lane == 0) trace[(size_t)blockIdx.x * 64 + 39] = (unsigned long long)w_spin;
        }
    } else if (warp == 8) {
        // ===== chunk loader / storer (fuse, lane 0): TMA-loads this CTA's
        // chunks ([cc][64] fp32 boxes of NCHW) into tnb buffers, TMA-stores
        // each converted [64][cc] tile into the NHWC workspace, refills a
        // buffer once its store has read it, and reports landed stores
        // (kPubLag behind) to the publisher.  Chunk coordinates come
        // pre-decoded from the ring (no divisions on this thread). =====
        if (FUSE && lane == 0 && n_my > 0) {
            constexpr int kPubLag = 1, kReport = 2;   // completion checked + reported every kReport chunks
            const uint32_t buf_bytes = (uint32_t)p.cc * 256;
            unsigned long long* tr = trace ? trace + (size_t)blockIdx.x * 64 : nullptr;
            long long c_conv = 0, c_rd = 0, c_pub = 0, c_dec = 0;
            if (tr) tr[58] = globaltimer_ns();
            auto entry = [&](int k) -> int4 {          // waits until the converters decoded chunk k
                if (ld_acquire_cta_smem(dec_ctr) <= k) {
                    const long long t0 = clock64();
                    while (ld_acquire_cta_smem(dec_ctr) <= k) {
                        if (clock64() - t0 > 8000000000ll) __trap();   // this wait, ~4 s
                    }
                    if (tr) c_dec += clock64() - t0;
                }
                return lds_int4(&cring[k & (kRing - 1)]);
            };
            auto load = [&](int k) {
                const int4 e = entry(k);
                const int b = k % p.tnb;
                mbar_arrive_expect_tx(&tfull[b], buf_bytes);
                tma_load_3d(tbuf + (size_t)b * buf_bytes, &tmap_src, &tfull[b], e.z, e.w, e.y);
            };
            unsigned long long* t2 = trace ? trace + (size_t)(512 + blockIdx.x) * 64 : nullptr;
            for (int k = 0; k < p.tnb && k < n_my; ++k) {
                load(k);
                if (t2 && k == 0) t2[4] = globaltimer_ns();
            }
            for (int k = 0; k < n_my; ++k) {
                const int b = k % p.tnb;
                const long long t0 = tr ? clock64() : 0;
                mbar_wait(&tconv[b], (uint32_t)(k / p.tnb) & 1);
                if (t2 && k == 0) t2[0] = globaltimer_ns();
                if (tr) c_conv += clock64() - t0;
                const int4 e = lds_int4(&cring[k & (kRing - 1)]);
                tma_store_3d(&tmap_dst, tbuf + (size_t)b * buf_bytes, e.w, e.z, e.y);
                bulk_commit();
                const int kn = k - 1 + p.tnb;             // refill chunk k-1's buffer with chunk k-1+tnb
                if (k >= 1 && kn < n_my) {
                    const long long t1 = tr ? clock64() : 0;
                    bulk_wait_read<1>();
                    if (tr) c_rd += clock64() - t1;
                    load(kn);
                }
                if (k >= kPubLag && ((k - kPubLag) % kReport) == 0) {
                    const long long t3 = tr ? clock64() : 0;
                    bulk_wait<kPubLag>();                 // all but the newest kPubLag stores have landed
                    if (tr) c_pub += clock64() - t3;
                    fence_proxy_async_global();           // async-proxy writes -> generic flag release
                    st_release_cta_smem(done_ctr, k - kPubLag + 1);
                    if (t2 && k == kPubLag) t2[1] = globaltimer_ns();
                }
            }
            bulk_wait<0>();
            fence_proxy_async_global();
            st_release_cta_smem(done_ctr, n_my);
            if (tr) {
                tr[33] = (unsigned long long)n_my;
                tr[34] = (unsigned long long)c_conv;
                tr[35] = (unsigned long long)c_rd;
                tr[36] = (unsigned long long)c_pub;
                tr[37] = (unsigned long long)c_dec;
                tr[38] = globaltimer_ns();
            }
        }
        __syncwarp();
    } else if (warp < 4 && !PROMOTE) {
        // ===== chunk converters + decoders (fuse): decode the chunk ring
        // one block ahead (parallel binary searches, no divisions on the
        // storer), then convert + transpose every loaded chunk in place
        // (RNE bf16 / RNA tf32) into the row-swizzled staging tile the
        // storer's TMA store expects. =====
        if (FUSE && n_my > 0) {
            const int tid = threadIdx.x;                  // 0..127
            const int w = (int)blockIdx.x, W = (int)gridDim.x;
            const uint32_t buf_bytes = (uint32_t)p.cc * 256;
            auto decode_block = [&](int k0) {             // chunks [k0, k0 + kDecode) -> ring
                if (tid < kDecode && k0 + tid < n_my)
                    cring[(k0 + tid) & (kRing - 1)] = chunk_decode(p, p.seq0 + w + (k0 + tid) * W);
                named_bar_sync(1, 128);
                if (tid == 0) st_release_cta_smem(dec_ctr, min(k0 + kDecode, n_my));
            };
            decode_block(0);
            if (kDecode < n_my) decode_block(kDecode);
            if (trace && tid == 0) trace[(size_t)(512 + blockIdx.x) * 64 + 3] = globaltimer_ns();
            for (int k = 0; k < n_my; ++k) {
                const int b = k % p.tnb;
                // one block ahead: decode chunks [k + 2 kDecode, ...) once the
                // publisher is past the ring slots they reuse
                if ((k % kDecode) == 0 && k + 2 * kDecode < n_my) {
                    const int k0 = k + 2 * kDecode;
                    if (tid == 0) {
                        const long long t0 = clock64();
                        while (ld_acquire_cta_smem(pub_ctr) < k0 + kDecode - kRing) {
                            __nanosleep(64);
                            if (clock64() - t0 > 8000000000ll) __trap();
                        }
                    }
                    named_bar_sync(1, 128);
                    decode_block(k0);
                }
                mbar_wait_sleep(&tfull[b], (uint32_t)(k / p.tnb) & 1, 32);
                uint8_t* buf = tbuf + (size_t)b * buf_bytes;
                float v[16];
                chunk_read(reinterpret_cast<const float*>(buf), p.cc, tid, v);
                named_bar_sync(1, 128);                   // every read of buf done
                chunk_write<BF16>(buf, p.cc, tid, v);
                fence_proxy_async_smem();                 // generic smem writes -> TMA store
                __syncwarp();
                if (lane == 0) mbar_arrive(&tconv[b]);
            }
        }
    } else if (PROMOTE && warp < 8) {
        // ===== promoted epilogue (8 warps; warp w: TMEM lane quadrant w % 4,
        // column half w / 4): each chunk's accumulator is added to fp32
        // registers with IEEE round-to-nearest adds, then released to the MMA
        // warp; after the tile's last chunk the registers go to NCHW Out =====
        constexpr int HB = BN / 2;
        const int q = warp & 3, half = warp >> 2;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int wi = unit; wi < p.num_work; wi += nunits) {
            // this work item's stages (split-K: its k range) in promotion chunks
            const int tile_w = SPLIT ? wi / p.splits : wi;
            const int it_beg = SPLIT ? (wi - tile_w * p.splits) * p.kper : 0;
            const int iters = SPLIT ? (min(p.k_iters, it_beg + p.kper) - it_beg) / p.kbs : p.k_iters / p.kbs;
            const int nchunk = (iters + p.pchunk - 1) / p.pchunk;
            float run[HB];
#pragma unroll
            for (int j = 0; j < HB; ++j) run[j] = 0.0f;
            for (int c = 0; c < nchunk; ++c) {
                mbar_wait_sleep(&tmem_full[acc], acc_phase, 64);
                tc_fence_after();
                const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + half * HB);
                // narrow loads at BN >= 192: the BN/2 sums + the load buffer
                // must stay within the 168 registers of a 384-thread CTA
                constexpr int LW = HB > 64 ? 8 : 16;
#pragma unroll
                for (int j0 = 0; j0 < HB; j0 += LW) {
                    uint32_t v[LW];
                    if constexpr (LW == 8) tmem_ld_32x32b_x8(t0 + (uint32_t)j0, v);
                    else tmem_ld_32x32b_x16(t0 + (uint32_t)j0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < LW; ++j) run[j0 + j] = __fadd_rn(run[j0 + j], __uint_as_float(v[j]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_leader(&tmem_empty[acc]);
                    else mbar_arrive(&tmem_empty[acc]);
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
            if constexpr (SPLIT) {
                // split-K (CG = 1, one wave): the promoted partial of this
                // k range -> its slab ([BN][128] column-major, as
                // store_partial), then warps 4-7 run the common arrival /
                // split-order reduction below
                float* slab = p.part + (size_t)wi * (kBM * BN) + q * 32 + lane;
#pragma unroll
                for (int j = 0; j < HB; ++j) __stcg(slab + (size_t)(half * HB + j) * kBM, run[j]);
                __threadfence();
                named_bar_sync(2, 256);
                if (warp < 4) continue;
                const int sp = wi - tile_w * p.splits;
                const int c_lo = BN * sp / p.splits, c_hi = BN * (sp + 1) / p.splits;
                float* red = reinterpret_cast<float*>(smem);
                if (warp == 4 && lane == 0) {
                    int* ctr = p.tile_ctr + tile_w;
                    atomicAdd(ctr, 1);
                    const long long t0 = clock64();
                    while (ld_acquire_gpu(ctr) < p.splits) {
                        __nanosleep(32);
                        if (clock64() - t0 > 8000000000ll) __trap();
                    }
                    fence_proxy_async_global();
                    const uint32_t bytes = (uint32_t)(c_hi - c_lo) * kBM * 4;
                    mbar_arrive_expect_tx(last_full, bytes * p.splits);
                    const float* src = p.part + (size_t)tile_w * p.splits * (kBM * BN) + (size_t)c_lo * kBM;
                    for (int s2 = 0; s2 < p.splits; ++s2)
                        bulk_load_g2s(red + (size_t)s2 * (c_hi - c_lo) * kBM, src + (size_t)s2 * (kBM * BN), bytes,
                                      last_full);
                }
                mbar_wait(last_full, 0);
                reduce_share<BN>(p, tile_w, red, c_lo, c_hi, warp & 3, lane);
                continue;
            }
            // registers -> NCHW Out (32 consecutive pixels of one (n, k) plane per warp store)
            const int tile = wi;
            const int m_tile = tile / p.num_n_tiles;
            const int n_tile = tile - m_tile * p.num_n_tiles;
            const int m = m_tile * (kBM * CG) + (int)rank * kBM + q * 32 + (int)lane;
            if (m < p.M) {
                const int img = m / p.HW, pix = m - img * p.HW;
                const int kbase = n_tile * BN + half * HB;
                float* obase = p.out + ((int64_t)img * p.K) * p.HW + pix;
#pragma unroll
                for (int j = 0; j < HB; ++j)
                    if (kbase + j < p.K) __stcs(obase + (int64_t)(kbase + j) * p.HW, run[j]);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===== epilogue: TMEM -> registers -> NCHW Out =====
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int wi = unit; wi < p.num_work; wi += nunits) {
            const int tile = SPLIT ? wi / p.splits : wi;
            mbar_wait_sleep(&tmem_full[acc], acc_phase, 256);
            tc_fence_after();
            if constexpr (SPLIT) {
                // (CG = 1, one wave: one work item per CTA, so the pipeline's
                // smem is idle now and every split of the tile is resident)
                store_partial<BN, 1>(p, tmem_base, wi, acc, 0, warp & 3, lane);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tmem_empty[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                const int sp = wi - tile * p.splits;
                const int c_lo = BN * sp / p.splits, c_hi = BN * (sp + 1) / p.splits;
                float* red = reinterpret_cast<float*>(smem);
                __threadfence();                          // this thread's slab stores -> GPU scope
                named_bar_sync(2, 128);
                if (warp == 4 && lane == 0) {
                    // arrive on the tile's counter, wait for its other splits,
                    // then bulk-copy this split's column share of every slab
                    int* ctr = p.tile_ctr + tile;
                    atomicAdd(ctr, 1);
                    const long long t0 = clock64();
                    while (ld_acquire_gpu(ctr) < p.splits) {
                        __nanosleep(32);
                        if (clock64() - t0 > 8000000000ll) __trap();
                    }
                    fence_proxy_async_global();           // other CTAs' generic stores -> bulk-copy reads
                    const uint32_t bytes = (uint32_t)(c_hi - c_lo) * kBM * 4;
                    mbar_arrive_expect_tx(last_full, bytes * p.splits);
                    const float* src = p.part + (size_t)tile * p.splits * (kBM * BN) + (size_t)c_lo * kBM;
                    for (int s2 = 0; s2 < p.splits; ++s2)
                        bulk_load_g2s(red + (size_t)s2 * (c_hi - c_lo) * kBM, src + (size_t)s2 * (kBM * BN), bytes,
                                      last_full);
                }
                mbar_wait(last_full, 0);
                reduce_share<BN>(p, tile, red, c_lo, c_hi, warp & 3, lane);
                continue;
            }
            const int ti_e = (wi - unit) / nunits;
            if (trace && warp == 4 && lane == 0 && ti_e < 8) trace[(size_t)blockIdx.x * 64 + 40 + 2 * ti_e] = globaltimer_ns();
            // the CTA's last tile is split: warps 0-3 store columns [BN/2, BN)
            const bool last = kSplitLast && wi + nunits >= p.num_work;
            store_accumulator<BN, CG>(p, tmem_base, tile, acc, rank, warp & 3, lane, 0, last ? BN / 2 : BN);
            tc_fence_before();
            __syncwarp();
            if (trace && warp == 4 && lane == 0 && ti_e < 8) trace[(size_t)blockIdx.x * 64 + 41 + 2 * ti_e] = globaltimer_ns();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_leader(&tmem_empty[acc]);
                else mbar_arrive(&tmem_empty[acc]);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }

    // Warps 0-3 (after the transform, if any): the second half of the last
    // accumulator, so the exposed tail of the kernel is half an epilogue.
    if (kSplitLast && warp < 4 && unit < p.num_tiles) {
        const int n_my = (p.num_tiles - unit + nunits - 1) / nunits;
        const int ti = n_my - 1;
        mbar_wait_sleep(last_full, 0, 256);
        tc_fence_after();
        store_accumulator<BN, CG>(p, tmem_base, unit + ti * nunits, ti & 1, rank, warp & 3, lane, BN / 2, BN);
    }

    // Teardown: every MMA has retired (the epilogues consumed every
    // accumulator) before the TMEM is released.
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
        else tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------------------
// host side

TcLayout tc_layout(const Problem& pb, bool bf16) {
    TcLayout L;
    L.elem = bf16 ? 2 : 4;
    const int cbytes = pb.C * L.elem;
    int cp_bytes;
    if (cbytes <= 32) cp_bytes = 32;
    else if (cbytes <= 64) cp_bytes = 64;
    else cp_bytes = (cbytes + 127) / 128 * 128;
    L.Cp = cp_bytes / L.elem;
    L.sw = cp_bytes >= 128 ? 128 : cp_bytes;
    L.bkc = L.sw / L.elem;
    L.n_cblk = L.Cp / L.bkc;
    L.in_ws_bytes = (size_t)pb.N * pb.Hin() * pb.Win() * L.Cp * L.elem;
    L.ker_ws_bytes = (size_t)pb.K * pb.R * pb.S * L.Cp * L.elem;
    L.cc = L.bkc < 32 ? L.bkc : 32;
    L.nch = L.Cp / L.cc;
    L.hh = L.bkc / L.cc;
    const int64_t P = pb.Hin() * pb.Win();
    L.npch = (P + 63) / 64;
    L.coop_ok = (P % 4) == 0 && (int64_t)pb.N * L.npch * L.nch < (1ll << 30);
    L.flag_bytes = L.coop_ok ? 128 + (size_t)pb.N * L.npch * L.nch * sizeof(int) : 0;
    return L;
}

int tc_promote_kblocks(const TcLayout& L) {
    // env CONV_PROMOTE_PRODUCTS: the promotion interval (study knob)
    static const int products = [] {
        const char* e = getenv("CONV_PROMOTE_PRODUCTS");
        return e && atoi(e) > 0 ? atoi(e) : kPromoteProducts;
    }();
    return std::max(1, (products + L.bkc - 1) / L.bkc);
}

// pipeline ring + barrier block, then (fuse) the transform region at a
// 1024-B boundary: tnb fp32 [cc][64] chunk buffers (converted in place),
// tnb mbarriers and tnb chunk slots.
static size_t tc_pipe_bytes(const TcLayout& L, const TcTile& t) {
    const size_t a = (size_t)t.kbs * kBM * L.sw, b = (size_t)t.kbs * (t.bn / t.cg) * L.sw;
    // barriers: full/empty per stage, 2+2 accumulator, ready/last/slot/counters,
    // and the fused transform's 2 x kMaxTnb chunk barriers + decode counter
    return (size_t)t.stages * (a + b) + (2 * t.stages + 8 + 2 * kMaxTnb + 1) * 8 + 16;
}
size_t tc_transform_smem_bytes(const TcLayout& L, int tnb) {
    return (size_t)tnb * L.cc * 256 + kRing * 16;
}
size_t tc_smem_bytes(const TcLayout& L, const TcTile& t) {
    size_t s = tc_pipe_bytes(L, t);
    if (t.fuse) s = (s + 1023) / 1024 * 1024 + tc_transform_smem_bytes(L, t.tnb);
    return 1024 /*align slack*/ + s;
}

cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev, bool with_in,
                          const RepackFuse& fz);


struct TcMaps {
    CUtensorMap a, b, src, dst;   // src/dst only with fuse (copies of a/b otherwise)
};

template <int BN, bool BF16, int CG, int KSTEPS, bool SPLIT, bool FUSE, bool PROMOTE = false>
static cudaError_t launch_tc(const TcMaps& m, const TcParams& prm, size_t smem, int grid, cudaStream_t st) {
    auto kfn = conv_igemm_tcgen05<BN, BF16, CG, KSTEPS, SPLIT, FUSE, PROMOTE>;
    // Opt in to the largest dynamic smem once per instantiation and device.
    static SmemOptIn opt;
    if (cudaError_t e = opt.ensure(kfn, smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    static const int no_pdl = getenv("CONV_NO_PDL") ? 1 : 0;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL after the repack
    attr[1].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    // The fused transform's and split-K's CTAs wait on work other CTAs of
    // the grid do: all of them must be resident at once.  They are -- one CTA
    // per SM (smem and registers), grid <= SM count -- as long as no other
    // such grid holds part of the GPU: tc_run serialises these launches per
    // device (ResidentChain).  No cooperative launch is requested (ncu
    // cannot replay cooperative cluster launches); a starved wait traps
    // after ~4 s without progress (watchdog) instead of hanging.
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kfn, m.a, m.b, m.src, m.dst, prm);
}

template <bool BF16, int CG, int KSTEPS>
static cudaError_t launch_tc_bn(int bn, const TcMaps& m, const TcParams& prm, size_t smem, int grid, cudaStream_t st) {
    if (prm.splits > 1) {          // split-K kernels: CG = 1, BN <= 128, not fused (tc_split_ok)
        if constexpr (CG == 1) {
            if (prm.pchunk > 0) {      // FP32_TC: promoted partials
                if constexpr (BF16 && KSTEPS == 4) {
                    switch (bn) {
                        case 32: return launch_tc<32, true, 1, 4, true, false, true>(m, prm, smem, grid, st);
                        case 64: return launch_tc<64, true, 1, 4, true, false, true>(m, prm, smem, grid, st);
                        case 128: return launch_tc<128, true, 1, 4, true, false, true>(m, prm, smem, grid, st);
                        default: break;
                    }
                }
                return cudaErrorInvalidValue;
            }
            switch (bn) {
                case 32: return launch_tc<32, BF16, 1, KSTEPS, true, false>(m, prm, smem, grid, st);
                case 64: return launch_tc<64, BF16, 1, KSTEPS, true, false>(m, prm, smem, grid, st);
                case 128: return launch_tc<128, BF16, 1, KSTEPS, true, false>(m, prm, smem, grid, st);
                default: break;
            }
        }
        return cudaErrorInvalidValue;
    }
    // Promoted accumulation (FP32_TC): bf16 (the epilogue's 8 warps hold
    // BN/2 fp32 sums each), no split-K, no fused transform
    if (prm.pchunk > 0) {
        if constexpr (BF16 && KSTEPS == 4) {
            switch (bn) {
                case 32: return launch_tc<32, true, CG, 4, false, false, true>(m, prm, smem, grid, st);
                case 64: return launch_tc<64, true, CG, 4, false, false, true>(m, prm, smem, grid, st);
                case 128: return launch_tc<128, true, CG, 4, false, false, true>(m, prm, smem, grid, st);
                case 192: return launch_tc<192, true, CG, 4, false, false, true>(m, prm, smem, grid, st);
                case 256: return launch_tc<256, true, CG, 4, false, false, true>(m, prm, smem, grid, st);
                default: break;
            }
        }
        return cudaErrorInvalidValue;
    }
    // The fused transform is a separate instance: compiled into the common
    // kernel its (untaken) code cost every non-fused plan ~3 % (Table-1 sweep
    // 660.6 vs 642.7 us on one box) -- instructions are fetched cold after
    // each L2 flush.
    if (prm.fuse) {
        switch (bn) {
            case 32: return launch_tc<32, BF16, CG, KSTEPS, false, true>(m, prm, smem, grid, st);
            case 64: return launch_tc<64, BF16, CG, KSTEPS, false, true>(m, prm, smem, grid, st);
            case 128: return launch_tc<128, BF16, CG, KSTEPS, false, true>(m, prm, smem, grid, st);
            case 192: return launch_tc<192, BF16, CG, KSTEPS, false, true>(m, prm, smem, grid, st);
            case 256: return launch_tc<256, BF16, CG, KSTEPS, false, true>(m, prm, smem, grid, st);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (bn) {
        case 32: return launch_tc<32, BF16, CG, KSTEPS, false, false>(m, prm, smem, grid, st);
        case 64: return launch_tc<64, BF16, CG, KSTEPS, false, false>(m, prm, smem, grid, st);
        case 128: return launch_tc<128, BF16, CG, KSTEPS, false, false>(m, prm, smem, grid, st);
        case 192: return launch_tc<192, BF16, CG, KSTEPS, false, false>(m, prm, smem, grid, st);
        case 256: return launch_tc<256, BF16, CG, KSTEPS, false, false>(m, prm, smem, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool BF16, int CG>
static cudaError_t launch_tc_sw(int sw, int bn, const TcMaps& m, const TcParams& prm, size_t smem, int grid,
                                cudaStream_t st) {
    switch (sw) {
        case 128: return launch_tc_bn<BF16, CG, 4>(bn, m, prm, smem, grid, st);
        case 64: return launch_tc_bn<BF16, CG, 2>(bn, m, prm, smem, grid, st);
        case 32: return launch_tc_bn<BF16, CG, 1>(bn, m, prm, smem, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

static CUtensorMapSwizzle swizzle_for(int bytes) {
    return bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

static cudaError_t encode_maps(const Problem& pb, const TcLayout& L, const TcTile& t, bool bf16, const float* in,
                               void* in_ws, void* ker_ws, TcMaps& m, std::string& err) {
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMapSwizzle swz = swizzle_for(L.sw);
    {
        // In NHWC: dims (C, W, H, N) innermost first.
        const int ac = L.a_chan ? L.a_chan : L.Cp;          // channels per pixel of the workspace
        cuuint64_t dims[4] = {(cuuint64_t)ac, (cuuint64_t)pb.Win(), (cuuint64_t)pb.Hin(), (cuuint64_t)pb.N};
        cuuint64_t strides[3] = {(cuuint64_t)ac * L.elem, (cuuint64_t)ac * L.elem * pb.Win(),
                                 (cuuint64_t)ac * L.elem * pb.Win() * pb.Hin()};
        // Bounding box per image: w in [-pw, Win-1+pw-D(S-1)], h likewise
        // (the window origins; with padding they start outside the tensor,
        // whose out-of-bounds elements TMA fills with zeros); the traversal
        // steps U pixels (elementStrides), so it visits exactly the origins
        // U*w - pw, U*h - ph of the output pixels, row by row, image by
        // image; tap (r, s) is the per-load im2col offset (D*s, D*r).
        int lower[2] = {-pb.pw, -pb.ph};
        int upper[2] = {pb.pw - pb.D * (pb.S - 1), pb.ph - pb.D * (pb.R - 1)};
        cuuint32_t estr[4] = {1, (cuuint32_t)pb.U, (cuuint32_t)pb.U, 1};
        CUresult r = g_encode_im2col(&m.a, dt, 4, in_ws, dims, strides, lower, upper, (cuuint32_t)L.bkc,
                                     (cuuint32_t)kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")"; return cudaErrorInvalidValue; }
    }
    {
        // Ker KRSC as 2-D [K rows][R*S*Cp cols].
        cuuint64_t dims[2] = {(cuuint64_t)pb.R * pb.S * L.Cp, (cuuint64_t)pb.K};
        cuuint64_t strides[1] = {(cuuint64_t)pb.R * pb.S * L.Cp * L.elem};
        cuuint32_t box[2] = {(cuuint32_t)L.bkc, (cuuint32_t)(t.bn / t.cg)};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = g_encode_tiled(&m.b, dt, 2, ker_ws, dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"; return cudaErrorInvalidValue; }
    }
    if (!t.fuse) {
        m.src = m.a;
        m.dst = m.b;
        return cudaSuccess;
    }
    const int64_t P = pb.Hin() * pb.Win();
    {
        // In NCHW fp32 as {P, C, N}; box = 64 pixels x cc channels; channels
        // >= C and pixels >= P are zero-filled (that is the Cp padding).
        cuuint64_t dims[3] = {(cuuint64_t)P, (cuuint64_t)pb.C, (cuuint64_t)pb.N};
        cuuint64_t strides[2] = {(cuuint64_t)P * 4, (cuuint64_t)P * 4 * pb.C};
        cuuint32_t box[3] = {64, (cuuint32_t)L.cc, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = g_encode_tiled(&m.src, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeTiled (In NCHW) failed (" + std::to_string((int)r) + ")"; return cudaErrorInvalidValue; }
    }
    {
        // workspace NHWC as {Cp, P, N}; box = cc channels x 64 pixels, swizzled
        // like the staging tile; stores past the image's last pixel are clipped
        cuuint64_t dims[3] = {(cuuint64_t)L.Cp, (cuuint64_t)P, (cuuint64_t)pb.N};
        cuuint64_t strides[2] = {(cuuint64_t)L.Cp * L.elem, (cuuint64_t)L.Cp * L.elem * P};
        cuuint32_t box[3] = {(cuuint32_t)L.cc, 64, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        CUresult r = g_encode_tiled(&m.dst, dt, 3, in_ws, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    swizzle_for(L.cc * L.elem), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeTiled (NHWC store) failed (" + std::to_string((int)r) + ")"; return cudaErrorInvalidValue; }
    }
    return cudaSuccess;
}

int tc_split_kper(const Problem& pb, const TcLayout& L, const TcTile& t) {
    const int k_iters = pb.R * pb.S * L.n_cblk;
    if (t.splits <= 1) return k_iters;
    const int stages = k_iters / t.kbs;
    const int per = (stages + t.splits - 1) / t.splits;       // stages per split
    if ((t.splits - 1) * per >= stages) return 0;             // the last split would be empty
    return per * t.kbs;
}

size_t tc_split_bytes(const Problem& pb, const TcLayout& L, const TcTile& t) {
    (void)L;
    if (t.splits <= 1) return 0;
    const int64_t tiles = ((pb.M() + 127) / 128) * ((pb.K + t.bn - 1) / t.bn);
    const size_t ctr = ((size_t)tiles * sizeof(int) + 255) / 256 * 256;
    return ctr + (size_t)tiles * t.splits * 128 * t.bn * sizeof(float);
}

bool tc_split_ok(const Problem& pb, const TcLayout& L, const TcTile& t) {
    if (t.splits <= 1) return true;
    if (t.fuse || t.cg != 1 || t.bn > 128 || t.splits > 16 || tc_split_kper(pb, L, t) == 0) return false;
    // the reduction stages `splits` column shares of <= ceil(BN/splits) columns
    // x 128 rows fp32 in the (then idle) pipeline shared memory
    const size_t share = (size_t)((t.bn + t.splits - 1) / t.splits) * 128 * 4;
    return (size_t)t.splits * share <= tc_pipe_bytes(L, t);
}

// Plans whose main kernel needs all of its CTAs resident at once (the fused
// transform waits on chunks other CTAs convert, split-K on the tile's other
// splits) are serialised per device across streams and host threads: each
// such conv_run waits (on the device) for the previous one's main kernel and
// records the device's chain event after its own.  Two such grids sharing
// the GPU could otherwise each hold part of the SMs and wait on CTAs that can
// never be scheduled.  Inside CUDA-graph capture the chain is not used (a
// captured stream cannot wait on an event recorded outside the capture): the
// graph's own order serialises its launches (include/conv.h).
struct ResidentChain {
    std::mutex mu;
    cudaEvent_t ev[kMaxDevices] = {};
};
static ResidentChain g_chain;

cudaError_t tc_run(const Problem& pb, const TcLayout& L, const TcTile& t, bool bf16,
                   const float* in, const float* ker, float* out, void* in_ws, void* ker_ws, void* flag_ws,
                   cudaStream_t st, int num_sms, cudaEvent_t* ev, std::string& err, const Problem* expand_src,
                   int split_pairs) {
    if (t.halo) {                          // the single-launch halo kernel (halo.cu)
        if (expand_src || split_pairs) { err = "the halo kernel runs plain problems only"; return cudaErrorInvalidValue; }
        return halo_run(pb, bf16, in, ker, out, ker_ws, st, ev, err);
    }
    if (expand_src && !split_pairs && (t.fuse || t.splits > 1)) { err = "tap-expanded plans run without the fused transform and split-K"; return cudaErrorInvalidValue; }
    if (split_pairs && (!expand_src || !bf16 || t.fuse)) {
        err = "FP32_TC plans run the promoted bf16 kernel: no fused transform";
        return cudaErrorInvalidValue;
    }
    if (t.fuse && (!L.coop_ok || !flag_ws)) { err = "fused transform needs a TMA-legal NCHW plane and flag workspace"; return cudaErrorInvalidValue; }
    // Tensor maps depend on the workspace (and, fused, In) addresses, known
    // only here; they are encoded on first use and cached.
    struct Key {
        const void* ws; const void* kws; const void* in; Problem pb; int bn; int cg; int kbs; int bf16; int fuse; int dev;
    };
    struct Entry { Key k; TcMaps m; };
    static std::mutex mu;
    static Entry cache[32];
    static int n_cached = 0, next_slot = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{in_ws, ker_ws, t.fuse ? (const void*)in : nullptr, pb, t.bn, t.cg, t.kbs, bf16 ? 1 : 0, t.fuse, dev};
    auto same = [&](const Key& a) {
        return a.ws == key.ws && a.kws == key.kws && a.in == key.in && memcmp(&a.pb, &key.pb, sizeof(Problem)) == 0 &&
               a.bn == key.bn && a.cg == key.cg && a.kbs == key.kbs && a.bf16 == key.bf16 && a.fuse == key.fuse &&
               a.dev == key.dev;
    };
    TcMaps maps;
    bool hit = false;
    {
        std::lock_guard<std::mutex> g(mu);
        for (int i = 0; i < n_cached; ++i)
            if (same(cache[i].k)) { maps = cache[i].m; hit = true; break; }
    }
    if (!hit) {
        cudaError_t e = encode_maps(pb, L, t, bf16, in, in_ws, ker_ws, maps, err);
        if (e != cudaSuccess) return e;
        std::lock_guard<std::mutex> g(mu);
        cache[next_slot] = Entry{key, maps};
        next_slot = (next_slot + 1) % 32;
        if (n_cached < 32) ++n_cached;
    }

    int* flags = t.fuse ? static_cast<int*>(flag_ws) + 32 : nullptr;
    const int n_flags = t.fuse ? (int)(pb.N * L.npch * L.nch) : 0;
    cudaError_t e = cudaSuccess;

    TcParams prm;
    memset(&prm, 0, sizeof(prm));
    prm.out = out;
    prm.M = (int)pb.M();
    prm.HW = pb.H * pb.W;
    prm.W = pb.W;
    prm.K = pb.K;
    prm.R = pb.R;
    prm.S = pb.S;
    prm.U = pb.U;
    prm.D = pb.D;
    prm.ph = pb.ph;
    prm.pw = pb.pw;
    prm.Cp = L.Cp;
    prm.bkc = L.bkc;
    prm.n_cblk = L.n_cblk;
    prm.k_iters = pb.R * pb.S * L.n_cblk;
    prm.num_n_tiles = (pb.K + t.bn - 1) / t.bn;
    const int tile_m = kBM * t.cg;
    const int num_m_tiles = (int)((pb.M() + tile_m - 1) / tile_m);
    prm.num_tiles = num_m_tiles * prm.num_n_tiles;
    prm.splits = t.splits > 1 ? t.splits : 1;
    prm.kper = tc_split_kper(pb, L, t);
    prm.num_work = prm.num_tiles * prm.splits;
    if (prm.splits > 1) {
        if (!tc_split_ok(pb, L, t) || !flag_ws || prm.num_work > num_sms) {
            err = "split-K needs fuse=0, cg=1, bn<=128, a split workspace, non-empty stage-aligned splits and one wave";
            return cudaErrorInvalidValue;
        }
        prm.tile_ctr = static_cast<int*>(flag_ws);
        prm.part = reinterpret_cast<float*>(static_cast<uint8_t*>(flag_ws) +
                                            ((size_t)prm.num_tiles * sizeof(int) + 255) / 256 * 256);
    }

    prm.stages = t.stages;
    prm.kbs = t.kbs;
    // FP32_TC: promote every ~kPromoteProducts products per output (9 k-blocks
    // of 64 channels = one 3x3 window of a channel block), R16
    prm.pchunk = split_pairs ? std::max(1, (tc_promote_kblocks(L) + t.kbs - 1) / t.kbs) : 0;
    const bool compact = split_pairs && L.a_chan && L.a_chan != L.Cp;
    if (compact) {
        const SplitPairs sp = conv::split_pairs(split_pairs);
        prm.pnb = split_cq(expand_src->C) / L.bkc;
        for (int i = 0; i < kSplitMaxPairs; ++i) prm.pip[i] = sp.ip[i];
    }
    prm.sw = (uint32_t)L.sw;
    prm.a_stage_bytes = (uint32_t)(t.kbs * kBM * L.sw);
    prm.b_stage_bytes = (uint32_t)(t.kbs * (t.bn / t.cg) * L.sw);
    const int units = num_sms / t.cg;
    const int grid = (prm.num_work < units ? prm.num_work : units) * t.cg;
    const size_t smem = tc_smem_bytes(L, t);
    prm.fuse = t.fuse;
    if (t.fuse) {
        prm.flags = flags;
        prm.in = in;
        prm.in_ws = in_ws;
        prm.C = pb.C;
        prm.P = (int)(pb.Hin() * pb.Win());
        prm.Win = (int)pb.Win();
        prm.Hin = (int)pb.Hin();
        prm.npch = (int)L.npch;
        prm.cc = L.cc;
        prm.nch = L.nch;
        prm.hh = L.hh;
        const int nunits = grid / t.cg;
        const int n_waves = (prm.num_tiles + nunits - 1) / nunits;
        prm.total_chunks = n_flags;
        prm.hh_log2 = L.hh == 2 ? 1 : 0;
        // group boundaries: the end (+1) of the input chunk-pixel range the
        // tiles of waves 0..w read; with more than 32 waves, consecutive
        // waves are merged (the order is a schedule heuristic only)
        const int per = (n_waves + 31) / 32;
        prm.n_groups = 0;
        for (int w = per - 1;; w += per) {
            const int wl = w < n_waves ? w : n_waves - 1;
            const int last_tile = std::min((wl + 1) * nunits, prm.num_tiles) - 1;
            const int m_tile = last_tile / prm.num_n_tiles;
            const int m1 = (int)std::min<int64_t>((int64_t)(m_tile + 1) * tile_m, pb.M()) - 1;
            const int n = m1 / prm.HW;
            const int h = (m1 - n * prm.HW) / prm.W;
            const int64_t rb = std::min<int64_t>(std::max<int64_t>(h * pb.U - pb.ph + pb.D * (pb.R - 1), 0), pb.Hin() - 1);
            int e = n * (int)L.npch + (int)((rb * pb.Win() + pb.Win() - 1) / 64) + 1;
            if (prm.n_groups > 0 && e < prm.gend[prm.n_groups - 1]) e = prm.gend[prm.n_groups - 1];
            prm.gend[prm.n_groups++] = e;
            if (wl == n_waves - 1) break;
        }
        prm.tnb = t.tnb;
        prm.tr_off = (uint32_t)((tc_pipe_bytes(L, t) + 1023) / 1024 * 1024);
    }

    // all-resident plans: serialise with the device's previous one (above)
    std::unique_lock<std::mutex> chain_lock;
    if (t.fuse || prm.splits > 1) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) { cudaGetLastError(); cs = cudaStreamCaptureStatusNone; }
        if (cs == cudaStreamCaptureStatusNone && dev >= 0 && dev < kMaxDevices) {
            chain_lock = std::unique_lock<std::mutex>(g_chain.mu);
            if (!g_chain.ev[dev] && cudaEventCreateWithFlags(&g_chain.ev[dev], cudaEventDisableTiming) != cudaSuccess) {
                err = "cannot create the all-resident chain event";
                return cudaErrorUnknown;
            }
            e = cudaStreamWaitEvent(st, g_chain.ev[dev], 0);
            if (e != cudaSuccess) { err = "cudaStreamWaitEvent (all-resident chain) failed"; return e; }
        }
    }

    RepackFuse fz;
    if (t.fuse) {
        fz.zero_ptr = static_cast<int*>(flag_ws);
        fz.zero_n = 32 + n_flags;
        fz.nch = L.nch;
        fz.cc = L.cc;
        // prologue = channels [0, pre_c) of group 0 (the chunk-pixels wave 0
        // reads), pre_c a multiple of 64 (the repack tile) and of bkc: in
        // sequence order that is the first pre_c / bkc channel blocks of group
        // 0, which the in-kernel transform then skips
        const int pre_c = std::min(L.Cp, (t.pre_c + 63) / 64 * 64);
        fz.pre_q = pre_c > 0 ? prm.gend[0] : 0;
        fz.pre_ch = pre_c / L.cc;
        prm.seq0 = (pre_c / L.bkc) * prm.gend[0] * L.hh;
    } else if (prm.splits > 1) {
        fz.zero_ptr = prm.tile_ctr;               // the repack launch clears the arrival counters
        fz.zero_n = prm.num_tiles;
    }
    if (split_pairs)
        e = launch_split(*expand_src, L.Cp, split_pairs, in, ker, in_ws, ker_ws, st, ev, fz.zero_ptr, fz.zero_n,
                         compact);
    else if (expand_src)
        e = launch_expand(*expand_src, L.Cp, bf16, in, ker, in_ws, ker_ws, st, ev);
    else
        e = launch_repack(pb, L.Cp, bf16, in, ker, in_ws, ker_ws, st, ev, /*with_in=*/!t.fuse, fz);
    if (e != cudaSuccess) { err = "repack launch failed"; return e; }

    static const char* trace_path = kTraceBuild ? getenv("CONV_TRACE") : nullptr;   // trace builds only
    static unsigned long long* trace_buf = nullptr;
    prm.trace = nullptr;
    if (trace_path) {
        if (!trace_buf) cudaMalloc(&trace_buf, 1024 * 64 * sizeof(unsigned long long));
        cudaMemsetAsync(trace_buf, 0, 1024 * 64 * sizeof(unsigned long long), st);
        prm.trace = trace_buf;
    }
    if (prm.k_iters % t.kbs != 0) { err = "k-blocks per stage must divide R*S*c-blocks"; return cudaErrorInvalidValue; }
    if (t.cg == 2)
        e = bf16 ? launch_tc_sw<true, 2>(L.sw, t.bn, maps, prm, smem, grid, st)
                 : launch_tc_sw<false, 2>(L.sw, t.bn, maps, prm, smem, grid, st);
    else
        e = bf16 ? launch_tc_sw<true, 1>(L.sw, t.bn, maps, prm, smem, grid, st)
                 : launch_tc_sw<false, 1>(L.sw, t.bn, maps, prm, smem, grid, st);
    if (e != cudaSuccess) { err = std::string("tcgen05 kernel launch failed: ") + cudaGetErrorString(e); return e; }
    if (chain_lock.owns_lock()) cudaEventRecord(g_chain.ev[dev], st);
    if (ev) cudaEventRecord(ev[2], st);
    if (prm.trace) {
        static unsigned long long host[1024 * 64];
        cudaStreamSynchronize(st);
        cudaMemcpy(host, prm.trace, sizeof(host), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(trace_path, "wb")) {
            fwrite(host, sizeof(unsigned long long), (size_t)1024 * 64, f);   // rows 512+: transform detail
            fclose(f);
        }
    }
    return cudaSuccess;
}

}  // namespace conv

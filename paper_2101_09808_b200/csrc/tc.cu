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
//   warps 0-3 (fuse = 1) In transform: NCHW fp32 -> NHWC rows of the next
//             channel block, one block ahead of the producer -> in_full[]
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

#include <atomic>
#include <mutex>

#include "internal.h"
#include "sm100.cuh"

namespace conv {

using namespace sm100;

static constexpr int kBM = 128;
static constexpr int kThreads = 384;        // 12 warps: TMA, MMA, alloc, -, 4 epilogue, 4 In-transform

struct TcParams {
    float* out;
    int M;            // N*H*W
    int HW;           // H*W
    int W;            // output width
    int K;            // output channels
    int R, S;
    int Cp, bkc, n_cblk;
    int k_iters;      // R*S*n_cblk
    int num_n_tiles;
    int num_tiles;
    int stages;
    int kbs;                  // k-blocks per pipeline stage (1, 2 or 4)
    uint32_t sw;              // 32 / 64 / 128 (bytes per operand row per k-block)
    uint32_t a_stage_bytes;   // kbs * 128 * sw
    uint32_t b_stage_bytes;   // kbs * (bn / cg) * sw
    uint32_t debug;           // experiments only (env CONV_DEBUG_MODE): 1 no MMA, 2 no TMA, 4 no stores
    unsigned long long* trace;  // experiments only (env CONV_TRACE): per-CTA timeline, 64 slots
    // fused In transform (a-3 inside the main kernel): NCHW fp32 -> NHWC workspace
    int fuse;                 // 1: warps 8-11 write the NHWC rows each tile needs; 0: workspace pre-filled
    const float* in;          // NCHW fp32 In
    void* in_ws;              // NHWC workspace (tf32-in-fp32 or bf16), [N][Hin][Win][Cp]
    int C, Hin, Win;
    int tap_outer;            // k order: 1 = (r, s, cb) [not with fuse], 0 = (cb, r, s)
};

// ---- fused NCHW -> NHWC transform of the input rows one tile needs ----------
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

// The rows of In (image n, input row h_in, all Win pixels, all Cp channels)
// read by the im2col loads of output pixels [m0, m0 + 128): for every image
// the tile touches, output rows h_lo..h_hi need input rows h_lo..h_hi+R-1.
// Work item = (row, VEC channels, 4 pixels) when the NCHW rows allow float4
// loads (Win % 4 == 0), else (row, VEC channels, 1 pixel); one 16-B store
// per pixel of VEC converted channels.  nthr threads starting at tid.
template <bool BF16>
__device__ void transform_tile_rows(const TcParams& p, int m0, int cbeg, int cend, int tid, int nthr) {
    constexpr int VEC = BF16 ? 8 : 4;
    constexpr int ES = BF16 ? 2 : 4;
    const int m1 = min(m0 + 128, p.M) - 1;
    if (m1 < m0) return;
    const int n_a = m0 / p.HW, n_b = m1 / p.HW;
    const bool vec4 = (p.Win & 3) == 0;
    const int pg = vec4 ? 4 : 1;
    const int groups = p.Win / pg;                 // pixel groups per row
    const int cvecs = (cend - cbeg) / VEC;
    const int per_row = groups * cvecs;
    const int64_t P = (int64_t)p.Hin * p.Win;
    for (int i0 = tid; i0 < per_row; i0 += nthr) {  // usually one (cv, g) per thread
        const int cv = i0 / groups;
        const int g = i0 - cv * groups;
        const int w0 = g * pg;
        const int c0 = cbeg + cv * VEC;
        for (int n = n_a; n <= n_b; ++n) {
            const int p_lo = n == n_a ? m0 - n * p.HW : 0;
            const int p_hi = n == n_b ? m1 - n * p.HW : p.HW - 1;
            const int h_lo = p_lo / p.W;
            const int h_hi = min(p_hi / p.W + p.R - 1, p.Hin - 1);
            const float* src = p.in + ((int64_t)n * p.C + c0) * P + (int64_t)h_lo * p.Win + w0;
            uint8_t* dst = reinterpret_cast<uint8_t*>(p.in_ws) +
                           ((((int64_t)n * p.Hin + h_lo) * p.Win + w0) * p.Cp + c0) * ES;
            const int64_t dst_row = (int64_t)p.Win * p.Cp * ES;
            for (int h = h_lo; h <= h_hi; ++h, src += p.Win, dst += dst_row) {
                float v[VEC][4];
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    if (c0 + j < p.C) {
                        const float* s = src + (int64_t)j * P;
                        if (vec4) {
                            const float4 x = __ldg(reinterpret_cast<const float4*>(s));
                            v[j][0] = x.x; v[j][1] = x.y; v[j][2] = x.z; v[j][3] = x.w;
                        } else {
                            v[j][0] = __ldg(s);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) v[j][q] = 0.0f;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (q < pg) {
                        uint4 o;
                        if (BF16) {
                            o.x = pack_bf16x2(v[0][q], v[1][q]);
                            o.y = pack_bf16x2(v[2][q], v[3][q]);
                            o.z = pack_bf16x2(v[4 % VEC][q], v[5 % VEC][q]);
                            o.w = pack_bf16x2(v[6 % VEC][q], v[7 % VEC][q]);
                        } else {
                            o.x = __float_as_uint(tf32_rna(v[0][q]));
                            o.y = __float_as_uint(tf32_rna(v[1][q]));
                            o.z = __float_as_uint(tf32_rna(v[2][q]));
                            o.w = __float_as_uint(tf32_rna(v[3][q]));
                        }
                        *reinterpret_cast<uint4*>(dst + (int64_t)q * p.Cp * ES) = o;
                    }
                }
            }
        }
    }
}

// CG = 1: one CTA per 128-pixel tile (tcgen05 cta_group::1, M = 128).
// CG = 2: a CTA pair (cluster of 2 on one TPC) per 256-pixel tile
//   (cta_group::2, M = 256): each CTA loads its own 128 A rows and HALF of
//   the BN B rows; the leader CTA issues the MMAs, which read both CTAs'
//   shared memory, and each CTA's TMEM receives its own 128 accumulator rows.
//   Per SM this halves the B operand traffic (L2 -> SMEM and SMEM -> tensor
//   core), which is what bounds the 1-CTA kernel on wide tiles.
template <int BN, bool BF16, int CG, int KSTEPS>
__global__ void __launch_bounds__(kThreads, 1)
conv_igemm_tcgen05(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + (size_t)p.stages * p.a_stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_b + (size_t)p.stages * p.b_stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + p.stages;
    uint64_t* tmem_full = bars + 2 * p.stages;
    uint64_t* tmem_empty = tmem_full + 2;
    uint64_t* in_full = tmem_empty + 2;           // fused In transform -> producer
    uint64_t* in_empty = in_full + 2;             // producer -> In transform (bounds run-ahead)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(in_empty + 2);

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
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4 * CG);    // one arrive per epilogue warp of the pair
            mbar_init(&in_full[i], 4);            // one arrive per transform warp
            mbar_init(&in_empty[i], 1);
        }
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
    const uint32_t wflavor = (p.debug >> 3) & 3;
    // Programmatic dependent launch: everything above overlapped the tail of
    // the repack launch; from here on the repacked workspace is read (and Out
    // written), so wait for the preceding grid to complete and flush.
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
            int u = 0, ue = 0;                            // (tile, channel block) units: waited / released
            for (int tile = unit; tile < p.num_tiles; tile += nunits) {
                const int m_tile = tile / p.num_n_tiles;
                const int n_tile = tile - m_tile * p.num_n_tiles;
                const int m0 = m_tile * (kBM * CG) + (int)rank * kBM;
                const int img = m0 / p.HW;
                const int pix = m0 - img * p.HW;
                const int h0 = pix / p.W;
                const int w0 = pix - h0 * p.W;
                const int kb0 = n_tile * BN + (int)rank * (BN / CG);   // this CTA's B rows
                const uint32_t a_blk = kBM * p.sw, b_blk = (BN / CG) * p.sw;
                // k iterations in a fixed order -- (cb, r, s) or (r, s, cb) --
                // tracked by counters (no divisions); a stage holds kbs
                // consecutive iterations, so the order does not depend on kbs.
                int cb = 0, r = 0, s = 0;
                for (int it0 = 0; it0 < p.k_iters; it0 += p.kbs) {
                    if (p.fuse) {   // channel blocks that start inside this stage must be written
                        int c2 = cb, r2 = r, s2 = s;
                        for (int kb = 0; kb < p.kbs; ++kb) {
                            if (r2 == 0 && s2 == 0) { mbar_wait(&in_full[u & 1], (u >> 1) & 1); ++u; }
                            if (++s2 == p.S) { s2 = 0; if (++r2 == p.R) { r2 = 0; ++c2; } }
                        }
                    }
                    const long long pw0 = p.trace ? clock64() : 0;
                    mbar_wait_flavor(&empty[stage], phase ^ 1, wflavor);
                    if (p.trace) prod_wait += clock64() - pw0;
                    uint8_t* a_dst = smem_a + (size_t)stage * p.a_stage_bytes;
                    uint8_t* b_dst = smem_b + (size_t)stage * p.b_stage_bytes;
                    const int cb_s = cb, r_s = r, s_s = s;
                    // advance the counters past this stage (all lanes, uniform)
                    for (int kb = 0; kb < p.kbs; ++kb) {
                        if (p.tap_outer) {
                            if (++cb == p.n_cblk) { cb = 0; if (++s == p.S) { s = 0; ++r; } }
                        } else {
                            if (++s == p.S) { s = 0; if (++r == p.R) { r = 0; ++cb; } }
                        }
                    }
                    if (elect_one_sync()) {
                        if (p.debug & 2) {
                            if (leader) mbar_arrive(&full[stage]);
                        } else {
                            if (leader) mbar_arrive_expect_tx(&full[stage], tx_bytes);
                            int c1 = cb_s, r1 = r_s, s1 = s_s;
                            for (int kb = 0; kb < p.kbs; ++kb) {
                                const int bx = (r1 * p.S + s1) * p.Cp + c1 * p.bkc;
                                if (CG == 2) {
                                    tma_load_im2col_4d_pair(a_dst + kb * a_blk, &tmap_a, &full[stage], c1 * p.bkc,
                                                            w0, h0, img, (uint16_t)s1, (uint16_t)r1, pol_a);
                                    tma_load_2d_pair(b_dst + kb * b_blk, &tmap_b, &full[stage], bx, kb0, pol_b);
                                } else {
                                    tma_load_im2col_4d(a_dst + kb * a_blk, &tmap_a, &full[stage], c1 * p.bkc,
                                                       w0, h0, img, (uint16_t)s1, (uint16_t)r1, pol_a);
                                    tma_load_2d(b_dst + kb * b_blk, &tmap_b, &full[stage], bx, kb0, pol_b);
                                }
                                if (p.tap_outer) {
                                    if (++c1 == p.n_cblk) { c1 = 0; if (++s1 == p.S) { s1 = 0; ++r1; } }
                                } else {
                                    if (++s1 == p.S) { s1 = 0; if (++r1 == p.R) { r1 = 0; ++c1; } }
                                }
                            }
                        }
                        if (p.fuse) {   // channel blocks that end inside this stage are consumed
                            int r2 = r_s, s2 = s_s, e2 = ue;
                            for (int kb = 0; kb < p.kbs; ++kb) {
                                if (r2 == p.R - 1 && s2 == p.S - 1) mbar_arrive(&in_empty[(e2++) & 1]);
                                if (++s2 == p.S) { s2 = 0; if (++r2 == p.R) r2 = 0; }
                            }
                        }
                    }
                    __syncwarp();
                    if (p.fuse) {   // same count in every lane (uniform)
                        int r2 = r_s, s2 = s_s;
                        for (int kb = 0; kb < p.kbs; ++kb) {
                            if (r2 == p.R - 1 && s2 == p.S - 1) ++ue;
                            if (++s2 == p.S) { s2 = 0; if (++r2 == p.R) r2 = 0; }
                        }
                    }
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                }
            }
            if (p.trace && lane == 0) {
                p.trace[(size_t)blockIdx.x * 64 + 60] = (unsigned long long)prod_wait;
                p.trace[(size_t)blockIdx.x * 64 + 61] = globaltimer_ns();
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
            const bool no_mma = (p.debug & 1) != 0;
            const int kbs = p.kbs;
            const int iters = p.k_iters / kbs;
            unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 64 : nullptr;
            int ti = 0;
            if (tr && lane == 0) tr[0] = globaltimer_ns();
            for (int tile = unit; tile < p.num_tiles; tile += nunits, ++ti) {
                mbar_wait_flavor(&tmem_empty[acc], acc_phase ^ 1, wflavor);
                tc_fence_after();
                if (tr && lane == 0 && ti < 8) tr[1 + 4 * ti] = globaltimer_ns();
                long long wait_cyc = 0;
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                uint32_t accum = 0;                      // first MMA of the tile overwrites D
                for (int it = 0; it < iters; ++it) {
                    const long long w0 = tr ? clock64() : 0;
                    mbar_wait_flavor(&full[stage], phase, wflavor);
                    if (tr) wait_cyc += clock64() - w0;
                    tc_fence_after();
                    if (elect_one_sync()) {
                        const uint64_t ad0 = a_desc0 + (uint64_t)(stage * a_step);
                        const uint64_t bd0 = b_desc0 + (uint64_t)(stage * b_step);
                        if (!no_mma) {
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
                // accumulator ready for the epilogue (of both CTAs)
                if (elect_one_sync()) {
                    if (CG == 2) tc_commit_pair_mc(&tmem_full[acc], 0x3);
                    else tc_commit(&tmem_full[acc]);
                }
                __syncwarp();
                if (tr && lane == 0 && ti < 8) {
                    tr[1 + 4 * ti + 1] = (unsigned long long)wait_cyc;
                    tr[1 + 4 * ti + 2] = globaltimer_ns();
                    tr[1 + 4 * ti + 3] = (unsigned long long)clock64();
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp < 4) {
        // ===== fused In transform: NCHW fp32 -> NHWC rows, one channel group
        // ahead of the producer =====
        if (p.fuse) {
            const int tid = threadIdx.x;
            int u = 0;
            for (int tile = unit; tile < p.num_tiles; tile += nunits) {
                const int m_tile = tile / p.num_n_tiles;
                // Every CTA writes the rows its own tiles read (tiles of other
                // CTAs may rewrite the same rows with the same values): the
                // only ordering needed is CTA-local.
                for (int cb = 0; cb < p.n_cblk; ++cb, ++u) {
                    mbar_wait_sleep(&in_empty[u & 1], ((u >> 1) & 1) ^ 1, 64);
                    transform_tile_rows<BF16>(p, m_tile * (kBM * CG) + (int)rank * kBM, cb * p.bkc,
                                              (cb + 1) * p.bkc, tid, 128);
                    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> TMA reads
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&in_full[u & 1]);
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===== epilogue: TMEM -> registers -> NCHW Out =====
        const int q = warp & 3;                       // TMEM lane quadrant of this warp
        const int row = q * 32 + (int)lane;           // accumulator row = pixel within the CTA's tile
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = unit; tile < p.num_tiles; tile += nunits) {
            const int m_tile = tile / p.num_n_tiles;
            const int n_tile = tile - m_tile * p.num_n_tiles;
            const int m = m_tile * (kBM * CG) + (int)rank * kBM + row;
            const int k0 = n_tile * BN;
            const bool valid_m = m < p.M;
            const int img = valid_m ? m / p.HW : 0;
            const int pix = valid_m ? m - img * p.HW : 0;
            float* obase = p.out + ((int64_t)img * p.K) * p.HW + pix;

            mbar_wait_sleep(&tmem_full[acc], acc_phase, 256);
            tc_fence_after();
            const int ti_e = (tile - unit) / nunits;
            if (p.trace && warp == 4 && lane == 0 && ti_e < 8) p.trace[(size_t)blockIdx.x * 64 + 40 + 2 * ti_e] = globaltimer_ns();
            const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
            for (int j0 = 0; j0 < BN; j0 += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(t0 + (uint32_t)j0, v);
                tmem_ld_wait();
                const int kbase = k0 + j0;
                if (valid_m && !(p.debug & 4)) {
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
            tc_fence_before();
            __syncwarp();
            if (p.trace && warp == 4 && lane == 0 && ti_e < 8) p.trace[(size_t)blockIdx.x * 64 + 41 + 2 * ti_e] = globaltimer_ns();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_leader(&tmem_empty[acc]);
                else mbar_arrive(&tmem_empty[acc]);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
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
    return L;
}

size_t tc_smem_bytes(const TcLayout& L, const TcTile& t) {
    const size_t a = (size_t)t.kbs * kBM * L.sw, b = (size_t)t.kbs * (t.bn / t.cg) * L.sw;
    return 1024 /*align slack*/ + (size_t)t.stages * (a + b) + (2 * t.stages + 8) * 8 + 16;
}

cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev, bool with_in);


template <int BN, bool BF16, int CG, int KSTEPS>
static cudaError_t launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& prm,
                             size_t smem, int grid, cudaStream_t st) {
    auto kfn = conv_igemm_tcgen05<BN, BF16, CG, KSTEPS>;
    // Opt in to the largest dynamic smem once per instantiation (per process).
    static std::atomic<int> smem_set{0};
    if (smem_set.load(std::memory_order_acquire) < (int)smem) {
        int optin = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
        if (e != cudaSuccess) return e;
        smem_set.store(optin, std::memory_order_release);
    }
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
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kfn, ta, tb, prm);
}

template <bool BF16, int CG, int KSTEPS>
static cudaError_t launch_tc_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                                const TcParams& prm, size_t smem, int grid, cudaStream_t st) {
    switch (bn) {
        case 32: return launch_tc<32, BF16, CG, KSTEPS>(ta, tb, prm, smem, grid, st);
        case 64: return launch_tc<64, BF16, CG, KSTEPS>(ta, tb, prm, smem, grid, st);
        case 128: return launch_tc<128, BF16, CG, KSTEPS>(ta, tb, prm, smem, grid, st);
        case 192: return launch_tc<192, BF16, CG, KSTEPS>(ta, tb, prm, smem, grid, st);
        case 256: return launch_tc<256, BF16, CG, KSTEPS>(ta, tb, prm, smem, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool BF16, int CG>
static cudaError_t launch_tc_sw(int sw, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                                const TcParams& prm, size_t smem, int grid, cudaStream_t st) {
    switch (sw) {
        case 128: return launch_tc_bn<BF16, CG, 4>(bn, ta, tb, prm, smem, grid, st);
        case 64: return launch_tc_bn<BF16, CG, 2>(bn, ta, tb, prm, smem, grid, st);
        case 32: return launch_tc_bn<BF16, CG, 1>(bn, ta, tb, prm, smem, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t tc_run(const Problem& pb, const TcLayout& L, const TcTile& t, bool bf16,
                   const float* in, const float* ker, float* out, void* in_ws, void* ker_ws,
                   cudaStream_t st, int num_sms, cudaEvent_t* ev, std::string& err) {
    const void* ws = in_ws;   // tensor-map cache key

    // Tensor maps depend on the workspace address, known only here; they are
    // encoded on first use and cached per (workspace, problem, tile).
    struct Key {
        const void* ws; const void* kws; Problem pb; int bn; int cg; int kbs; int bf16; int dev;  // (fuse does not change the maps)
    };
    struct Entry { Key k; CUtensorMap ta, tb; };
    static std::mutex mu;
    static Entry cache[16];
    static int n_cached = 0, next_slot = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{ws, ker_ws, pb, t.bn, t.cg, t.kbs, bf16 ? 1 : 0, dev};
    auto same = [&](const Key& a) {
        return a.ws == key.ws && a.kws == key.kws && memcmp(&a.pb, &key.pb, sizeof(Problem)) == 0 && a.bn == key.bn && a.cg == key.cg && a.kbs == key.kbs &&
               a.bf16 == key.bf16 && a.dev == key.dev;
    };
    CUtensorMap ta, tb;
    bool hit = false;
    {
        std::lock_guard<std::mutex> g(mu);
        for (int i = 0; i < n_cached; ++i)
            if (same(cache[i].k)) { ta = cache[i].ta; tb = cache[i].tb; hit = true; break; }
    }
    if (!hit) {
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMapSwizzle swz = L.sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : (L.sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    {
        // In NHWC: dims (C, W, H, N) innermost first.
        cuuint64_t dims[4] = {(cuuint64_t)L.Cp, (cuuint64_t)pb.Win(), (cuuint64_t)pb.Hin(), (cuuint64_t)pb.N};
        cuuint64_t strides[3] = {(cuuint64_t)L.Cp * L.elem, (cuuint64_t)L.Cp * L.elem * pb.Win(),
                                 (cuuint64_t)L.Cp * L.elem * pb.Win() * pb.Hin()};
        // Bounding box per image: w in [0, Win-1-(S-1)], h in [0, Hin-1-(R-1)]:
        // the traversal visits exactly the output pixels of valid conv.
        int lower[2] = {0, 0};
        int upper[2] = {-(pb.S - 1), -(pb.R - 1)};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = g_encode_im2col(&ta, dt, 4, in_ws, dims, strides, lower, upper, (cuuint32_t)L.bkc,
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
        CUresult r = g_encode_tiled(&tb, dt, 2, ker_ws, dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"; return cudaErrorInvalidValue; }
    }
    std::lock_guard<std::mutex> g(mu);
    cache[next_slot] = Entry{key, ta, tb};
    next_slot = (next_slot + 1) % 16;
    if (n_cached < 16) ++n_cached;
    }

    cudaError_t e = launch_repack(pb, L.Cp, bf16, in, ker, in_ws, ker_ws, st, ev, /*with_in=*/!t.fuse);
    if (e != cudaSuccess) { err = "repack launch failed"; return e; }

    TcParams prm;
    prm.out = out;
    prm.M = (int)pb.M();
    prm.HW = pb.H * pb.W;
    prm.W = pb.W;
    prm.K = pb.K;
    prm.R = pb.R;
    prm.S = pb.S;
    prm.Cp = L.Cp;
    prm.bkc = L.bkc;
    prm.n_cblk = L.n_cblk;
    prm.k_iters = pb.R * pb.S * L.n_cblk;
    prm.num_n_tiles = (pb.K + t.bn - 1) / t.bn;
    static const uint32_t debug_mode = [] {
        const char* e = getenv("CONV_DEBUG_MODE");
        return e ? (uint32_t)atoi(e) : 0u;
    }();
    prm.debug = debug_mode;
    prm.fuse = t.fuse;
    static const int env_order = [] { const char* e = getenv("CONV_KORDER"); return e ? atoi(e) : -1; }();
    // One order for every configuration (fused or not), so results are
    // bit-identical across tilings (P10); env CONV_KORDER=1 is for experiments.
    prm.tap_outer = t.fuse ? 0 : (env_order >= 0 ? env_order : 0);
    prm.in = in;
    prm.in_ws = in_ws;
    prm.C = pb.C;
    prm.Hin = (int)pb.Hin();
    prm.Win = (int)pb.Win();
    static const char* trace_path = getenv("CONV_TRACE");
    static unsigned long long* trace_buf = nullptr;
    prm.trace = nullptr;
    if (trace_path) {
        if (!trace_buf) cudaMalloc(&trace_buf, 1024 * 64 * sizeof(unsigned long long));
        cudaMemsetAsync(trace_buf, 0, 1024 * 64 * sizeof(unsigned long long), st);
        prm.trace = trace_buf;
    }
    const int tile_m = kBM * t.cg;
    const int num_m_tiles = (int)((pb.M() + tile_m - 1) / tile_m);
    prm.num_tiles = num_m_tiles * prm.num_n_tiles;
    prm.stages = t.stages;
    prm.kbs = t.kbs;
    prm.sw = (uint32_t)L.sw;
    prm.a_stage_bytes = (uint32_t)(t.kbs * kBM * L.sw);
    prm.b_stage_bytes = (uint32_t)(t.kbs * (t.bn / t.cg) * L.sw);
    const int units = num_sms / t.cg;
    const int grid = (prm.num_tiles < units ? prm.num_tiles : units) * t.cg;
    const size_t smem = tc_smem_bytes(L, t);
    if (prm.k_iters % t.kbs != 0) { err = "k-blocks per stage must divide R*S*c-blocks"; return cudaErrorInvalidValue; }
    if (t.cg == 2)
        e = bf16 ? launch_tc_sw<true, 2>(L.sw, t.bn, ta, tb, prm, smem, grid, st)
                 : launch_tc_sw<false, 2>(L.sw, t.bn, ta, tb, prm, smem, grid, st);
    else
        e = bf16 ? launch_tc_sw<true, 1>(L.sw, t.bn, ta, tb, prm, smem, grid, st)
                 : launch_tc_sw<false, 1>(L.sw, t.bn, ta, tb, prm, smem, grid, st);
    if (e != cudaSuccess) { err = std::string("tcgen05 kernel launch failed: ") + cudaGetErrorString(e); return e; }
    if (ev) cudaEventRecord(ev[2], st);
    if (prm.trace) {
        static unsigned long long host[1024 * 64];
        cudaStreamSynchronize(st);
        cudaMemcpy(host, prm.trace, sizeof(host), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(trace_path, "wb")) {
            fwrite(host, sizeof(unsigned long long), (size_t)grid * 64, f);
            fclose(f);
        }
    }
    return cudaSuccess;
}

}  // namespace conv

// simt.cu -- K4: FP32 SIMT direct convolution.
//
// Eq. 1 on native NCHW In with fp32 FFMA, no tensor cores.
// The structure follows the paper's own CPU design, re-targeted to an SM:
//   * packing (Sec. 6): Ker [K,C,R,S] -> [K/BKo, C, R, S, BKo]
//     so that a CTA's kernel slab is contiguous and a thread's TK output
//     channels are adjacent (vector loads, warp broadcast) -- the paper's
//     [K/VecLen, C, R, S, VecLen] with VecLen = BKo;
//   * outer-product register tile (Fig. 4 / Listing 4): each
//     thread holds TK output channels x TW output pixels of accumulators; per
//     (c, r, s) it loads TK kernel values (float4, broadcast) and TW input
//     values (one per pixel, conflict-free: the TW pixels of a thread are 32
//     apart, so a warp's loads are 32 consecutive pixels);
//   * shared-memory tile = Eq. 4's In + Ker footprints:
//     bc channels x tn images x (th+R-1) input rows x Win, plus
//     bc x R x S x BKo kernel values, double-buffered with cp.async;
//   * parallelism over non-reduction dims only: grid over
//     (image tile x row tile, k tile); the c,r,s reduction stays inside a
//     thread in a fixed order (c ascending, then r, then s).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"
#include "sm100.cuh"

namespace conv {

// Launch with programmatic stream serialization: the kernel's prologue
// overlaps the tail of the Ker packing grid; it calls griddepcontrol.wait
// before reading the packed kernel.
template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kfn, dim3 grid, int threads, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    static const int no_pdl = getenv("CONV_NO_PDL") ? 1 : 0;   // experiments
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, args...);
}

struct SimtParams {
    int N, K, C, H, W, R, S;
    int U;            // stride (v1 only): output (h, w) reads input rows U*h + r, columns U*w + s
    int Hin, Win, HW, RS;
    int tn, th, bc, kg;
    int bko;          // kg * TK
    int D;            // dilation (v1 only): tap (r, s) reads rows / columns D*r, D*s further
    int rows_in;      // (th - 1) * U + D * (R - 1) + 1
    int ph, pw;       // zero padding (v1 only): smem rows hold input rows h0*U - ph + i, columns c - pw
    int pitch;        // smem row pitch: Win + 2 * pw
    int plane;        // tn * rows_in * pitch  (floats per channel in smem)
    int n_htiles;     // ceil(H / th)
    int nchunks;      // ceil(C / bc)
    int cper;         // split-C: chunks per split (blockIdx.z), = nchunks without a split
    int64_t zstride;  // split-C: floats between the splits' partial outputs (0 without a split)
    int bp;           // tn * th * W (real pixels per CTA tile)
    int vec4_in;      // Win % 4 == 0
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Split-C: Out = the splits' partial outputs summed in split order 0..S-1
// (fixed, so the result is deterministic for a given split count).
__global__ void __launch_bounds__(256) reduce_splits(const float* __restrict__ part, float* __restrict__ out,
                                                     int64_t total, int S) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        float v = __ldcg(part + i);
        for (int z = 1; z < S; ++z) v += __ldcg(part + (int64_t)z * total + i);
        out[i] = v;
    }
}

// Packing kernel: Ker KCRS -> [ceil(K/bko)][C][R][S][bko], k >= K zero.
// k tile kb's source is ONE contiguous [bko][C*R*S] block of KCRS and its
// destination the contiguous [C*R*S][bko] block, so the pack is a transpose
// per k tile: a CTA stages a bko x cw slice (cw = 1024 / bko columns) in
// shared memory with coalesced row reads and writes it back with coalesced
// column-major stores.  (r02c: the per-element gather below it read each
// element from its own 32-B sector -- 1.1-1.3 TB/s on the large Table-1
// layers, 25 % of the Table-1 SIMT step time; tiled 16-B: Table-1 SIMT
// total 2329 -> 2042 us.)
__global__ void __launch_bounds__(256) pack_ker_simt_tiled(const float* __restrict__ ker, float* __restrict__ out,
                                                           int K, int CRS, int bko, int cw, int nchunk) {
    __shared__ float tile[1024 + 64];            // bko x (cw + 1), bko * cw = 1024
    const int kb = (int)blockIdx.x / nchunk;
    const int c0 = ((int)blockIdx.x - kb * nchunk) * cw;
    const int ncol = CRS - c0 < cw ? CRS - c0 : cw;
    const int pitch = cw + 1;                    // odd: the column reads hit distinct banks
    if ((CRS & 3) == 0) {
        // 16-B units both ways (CRS % 4 == 0: rows, c0 and the output block
        // are 16-B aligned; bko is a multiple of 4)
        const int cw4 = cw >> 2;
        for (int e = threadIdx.x; e < bko * cw4; e += blockDim.x) {
            const int r = e / cw4, j = (e - r * cw4) * 4;
            const int k = kb * bko + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < K && j < ncol) v = __ldg(reinterpret_cast<const float4*>(ker + (int64_t)k * CRS + c0 + j));
            float* t = tile + r * pitch + j;
            t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
        }
        __syncthreads();
        float4* o = reinterpret_cast<float4*>(out + ((int64_t)kb * CRS + c0) * bko);
        const int b4 = bko >> 2;
        for (int e = threadIdx.x; e < ncol * b4; e += blockDim.x) {
            const int j = e / b4, r = (e - j * b4) * 4;
            const float* t = tile + r * pitch + j;
            o[e] = make_float4(t[0], t[pitch], t[2 * pitch], t[3 * pitch]);
        }
    } else {
        for (int e = threadIdx.x; e < bko * cw; e += blockDim.x) {
            const int r = e / cw, j = e - r * cw;
            const int k = kb * bko + r;
            tile[r * pitch + j] = (k < K && j < ncol) ? __ldg(ker + (int64_t)k * CRS + c0 + j) : 0.0f;
        }
        __syncthreads();
        float* o = out + ((int64_t)kb * CRS + c0) * bko;
        for (int e = threadIdx.x; e < ncol * bko; e += blockDim.x) {
            const int j = e / bko, r = e - j * bko;
            o[e] = tile[r * pitch + j];
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");   // at the end of each CTA (see pack_ker_simt)
}

// (the r01-r02b per-element form, kept for the A/B: CONV_SIMT_PACK_GATHER=1)
__global__ void __launch_bounds__(256) pack_ker_simt(const float* __restrict__ ker, float* __restrict__ out,
                                                     int K, int C, int RS, int bko, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(i % bko);
        const int64_t t = i / bko;            // (kb*C + c)*RS + rs
        const int rs = (int)(t % RS);
        const int64_t t2 = t / RS;             // kb*C + c
        const int c = (int)(t2 % C);
        const int64_t kb = t2 / C;
        const int64_t k = kb * bko + kk;
        out[i] = k < K ? __ldg(ker + (k * C + c) * RS + rs) : 0.0f;
    }
    // Trigger the dependent SIMT launch only at the end of each CTA: triggered
    // at the start, the (small) SIMT grid was placed while this grid still
    // held most SMs and piled onto the few with room -- measured 2-3x slower
    // on the small Table-1 layers (R2 92 vs 33 us, M6 612 vs 199 us).
    asm volatile("griddepcontrol.launch_dependents;");
}

template <int TK, int TW, bool SPLITC>
__global__ void __launch_bounds__(512) conv_direct_simt(const float* __restrict__ in,
                                                         const float* __restrict__ kerp,
                                                         float* __restrict__ out, const SimtParams p) {
    extern __shared__ __align__(128) float sm[];
    const int in_stage = p.bc * p.plane;
    const int ker_stage = p.bc * p.RS * p.bko;
    const int stage_floats = in_stage + ker_stage;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int kgi = warp % p.kg;
    const int pwi = warp / p.kg;

    const int nt = blockIdx.x / p.n_htiles;
    const int ht = blockIdx.x - nt * p.n_htiles;
    const int n0 = nt * p.tn;
    const int h0 = ht * p.th;
    const int kb = blockIdx.y;
    const int k0 = kb * p.bko;

    // Per-slot pixel offsets into the smem In tile.
    int off[TW];
    int pix_img[TW], pix_h[TW], pix_w[TW];
    bool valid[TW];
    const int thw = p.th * p.W;
#pragma unroll
    for (int j = 0; j < TW; ++j) {
        const int q = pwi * 32 * TW + lane + 32 * j;
        const int img = q / thw;
        const int rem = q - img * thw;
        const int h = rem / p.W;
        const int w = rem - h * p.W;
        valid[j] = q < p.bp && (n0 + img) < p.N && (h0 + h) < p.H;
        off[j] = valid[j] ? (img * p.rows_in + h * p.U) * p.pitch + w * p.U : 0;
        pix_img[j] = img;
        pix_h[j] = h;
        pix_w[j] = w;
    }

    float acc[TK][TW];
#pragma unroll
    for (int i = 0; i < TK; ++i)
#pragma unroll
        for (int j = 0; j < TW; ++j) acc[i][j] = 0.0f;

    auto load_stage = [&](int buf, int chunk) {
        float* in_s = sm + buf * stage_floats;
        float* ker_s = in_s + in_stage;
        const int c0 = chunk * p.bc;
        // In: bc*tn segments of rows_in*pitch contiguous floats.
        const int seg_len = p.rows_in * p.pitch;
        for (int seg = 0; seg < p.bc * p.tn; ++seg) {
            const int cc = seg / p.tn;
            const int img = seg - cc * p.tn;
            const int c = c0 + cc;
            const int n = n0 + img;
            const bool seg_ok = c < p.C && n < p.N;
            const int hin0 = h0 * p.U - p.ph;     // first input row of the tile (< 0: padding)
            float* s = in_s + cc * p.plane + img * seg_len;
            if (p.ph | p.pw) {
                // zero padding: element (i, col) of the segment is input row
                // hin0 + i, column col - pw, or zero outside the input
                const float* gp = in + ((int64_t)n * p.C + c) * p.Hin * p.Win;
                for (int e = threadIdx.x; e < seg_len; e += blockDim.x) {
                    const int i = e / p.pitch, col = e - i * p.pitch - p.pw, gr = hin0 + i;
                    const bool ok = seg_ok && gr >= 0 && gr < p.Hin && col >= 0 && col < p.Win;
                    cp_async4(s + e, ok ? gp + (int64_t)gr * p.Win + col : in, ok);
                }
                continue;
            }
            const float* g = in + (((int64_t)n * p.C + c) * p.Hin + hin0) * p.Win;
            // valid elements: rows < Hin - hin0
            const int rows_ok = p.Hin - hin0 < p.rows_in ? p.Hin - hin0 : p.rows_in;
            const int len_ok = seg_ok ? rows_ok * p.Win : 0;
            if (p.vec4_in) {
                for (int e = threadIdx.x * 4; e < seg_len; e += blockDim.x * 4)
                    cp_async16(s + e, e < len_ok ? g + e : in, e < len_ok);
            } else {
                for (int e = threadIdx.x; e < seg_len; e += blockDim.x)
                    cp_async4(s + e, e < len_ok ? g + e : in, e < len_ok);
            }
        }
        // Ker: contiguous slab of the packed tensor, channels >= C zero.
        const int cvalid = p.C - c0 < p.bc ? p.C - c0 : p.bc;
        const int len_ok = cvalid * p.RS * p.bko;
        const float* g = kerp + (((int64_t)kb * p.C + c0) * p.RS) * p.bko;
        for (int e = threadIdx.x * 4; e < ker_stage; e += blockDim.x * 4)
            cp_async16(ker_s + e, e < len_ok ? g + e : kerp, e < len_ok);
    };

    asm volatile("griddepcontrol.wait;" ::: "memory");   // packed Ker written by the previous grid
    // split-C (separate instances, so the plain loop keeps its exact code --
    // the runtime range measured 3.5 % slower on the batched layer): this
    // CTA's channel chunks [c_beg, c_end) and its partial-output slab
    const int c_beg = SPLITC ? (int)blockIdx.z * p.cper : 0;
    const int c_end = SPLITC ? min(p.nchunks, c_beg + p.cper) : p.nchunks;
    if (SPLITC) out += (int64_t)blockIdx.z * p.zstride;
    load_stage(0, c_beg);
    cp_async_commit();
    for (int chunk = c_beg; chunk < c_end; ++chunk) {
        const int buf = (chunk - c_beg) & 1;
        if (chunk + 1 < c_end) load_stage(buf ^ 1, chunk + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const float* in_s = sm + buf * stage_floats;
        const float* ker_s = in_s + in_stage;
        const int cc_end = p.C - chunk * p.bc < p.bc ? p.C - chunk * p.bc : p.bc;
        for (int cc = 0; cc < cc_end; ++cc) {
            for (int r = 0; r < p.R; ++r) {
                const float* ip = in_s + cc * p.plane + r * p.D * p.pitch;
                const float* kp = ker_s + ((cc * p.R + r) * p.S) * p.bko + kgi * TK;
                for (int s = 0; s < p.S; ++s) {
                    float iv[TW];
#pragma unroll
                    for (int j = 0; j < TW; ++j) iv[j] = ip[off[j] + s * p.D];
                    float kv[TK];
#pragma unroll
                    for (int i = 0; i < TK; i += 4) {
                        const float4 k4 = *reinterpret_cast<const float4*>(kp + s * p.bko + i);
                        kv[i] = k4.x; kv[i + 1] = k4.y; kv[i + 2] = k4.z; kv[i + 3] = k4.w;
                    }
#pragma unroll
                    for (int i = 0; i < TK; ++i)
#pragma unroll
                        for (int j = 0; j < TW; ++j) acc[i][j] = fmaf(kv[i], iv[j], acc[i][j]);
                }
            }
        }
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < TK; ++i) {
        const int k = k0 + kgi * TK + i;
        if (k >= p.K) break;
#pragma unroll
        for (int j = 0; j < TW; ++j) {
            if (valid[j]) {
                const int64_t o = (((int64_t)(n0 + pix_img[j]) * p.K + k) * p.H + (h0 + pix_h[j])) * p.W + pix_w[j];
                out[o] = acc[i][j];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K4 v2: the paper's microkernel (Fig. 4) on an SM.  A thread
// owns TK output channels x TW CONSECUTIVE output pixels of one row; per (c, r)
// it loads the TW+S-1 input values of its window once (vector LDS from a
// row-padded shared-memory tile) and reuses them across the S taps in
// registers; per (c, r, s) the TK kernel values are a broadcast float4 load.
// FFMA : LDS = S*TK*TW : (ceil((TW+S-1)/4) + S*TK/4)  (96 : 8 at TK=8,TW=4,S=3).
struct Simt2Params {
    int N, K, C, H, W, R, S;
    int Hin, Win;
    int tn, th, bc, kg;
    int bko;          // kg * TK
    int rows_in;      // th + R - 1
    int pitch;        // floats per smem row (>= groups*TW + S - 1, multiple of 4)
    int istride;      // floats between the images in smem (cp.async layout: of one channel, >= rows_in * pitch;
                      //    TMA layout: an image's bc channels, bc * rows_in * pitch; simt2_layout)
    int cstride;      // floats between the channels of an image in smem (cp.async: tn * istride; TMA: rows_in * pitch)
    int plane;        // cp.async layout: tn * istride (floats per channel in smem)
    int in_stage;     // floats of one stage's In tile
    int lpi;          // lanes (pixel-group slots) per image: per_img, or rounded up to 8 in the TMA layout
                      //    so that no quarter-warp straddles two images (conflict-free window loads)
    int groups;       // ceil(W / TW): pixel groups per output row
    int n_htiles;
    int nchunks;
    int cper;         // split-C: chunks per split (blockIdx.z)
    int64_t zstride;  // split-C: floats between partial outputs
    int slots;        // tn * lpi (pixel-group slots per CTA)
    int stages;       // TMA layout: ring depth (<= kSimt2MaxStages)
    int ktiles;       // ceil(K / bko): grid x = (image tile, row tile) * ktiles + k tile -- the k
                      //    tiles of an image tile run together, so its In tile is read from HBM once
    int vec4;         // Win % 4 == 0: 16-B copies of input rows
    uint32_t tx_in;   // TMA layout: bytes of one In box (tn * bc * rows_box * pitch * 4)
    int flat;         // flat row mode (SimtTile::flat): grid x = slot tile * ktiles + k tile, slot tile
                      //    = 32*pw consecutive (image, row) slots; the box starts at the slot tile's
                      //    first image, smem [c][img][rows_box][pitch] (istride = rows_box * pitch)
    int solo;         // remainder launch (simt_rem_tiles; flat TMA tiles, TK = 1 instance): > 0 = CTAs per
                      //    (slot tile, k tile); CTA blockIdx is channels 4 * (blockIdx % solo) + warp of k tile
                      //    (blockIdx / solo) % ktiles of slot tile tile0 + blockIdx / (solo * ktiles)
    int tile0;        // remainder launch: first slot tile
    int trigger;      // griddepcontrol.launch_dependents once the packed Ker is complete
    int endwait;      // griddepcontrol.wait at the CTA's end (so that this grid's end implies the previous one's)
    int nowait;       // main grid launched behind the remainder grid: no griddepcontrol.wait (that would
                      //    wait for the remainder grid's end; the packed Ker was complete before the
                      //    remainder CTAs triggered this launch)
};

static constexpr int kSimt2Stages = 3;     // v2 shared-memory ring depth (cp.async layout; TMA default)
static constexpr int kSimt2MaxStages = 4;  // TMA layout: ring depth p.stages <= this
#ifndef CONV_SIMT_CC_UNROLL
#define CONV_SIMT_CC_UNROLL 0              // v2 channel-loop unroll for every instance (A/B builds; 0: the default below)
#endif
#ifndef CONV_SIMT_SHFL
#define CONV_SIMT_SHFL 2                   // TW = 4 halo by warp shuffle: 2 for TK = 8 tiles (default),
#endif                                     // 1 for every TW = 4 tile, 0 never (A/B builds)
#ifndef CONV_SIMT_FFMA2
#define CONV_SIMT_FFMA2 1                  // v2 inner product on FFMA2 (r02: 4 % slower with the cp.async
                                           // copies; r02b TMA layout: 1184-1194 vs 1207 us, 100 vs 114 registers)
#endif

// Row-mode TK = 8 instances hold 112 accumulators: at most 256 threads, so
// that ptxas may give a thread up to 255 registers.
template <int TK, int TW>
struct Simt2Threads { static constexpr int value = TK * TW > 64 ? 256 : 512; };

template <int TK, int TW, int KR, int KS, bool SPLITC, bool TMA>   // KR = 0: runtime R
__global__ void __launch_bounds__(Simt2Threads<TK, TW>::value) conv_direct_simt2(const float* __restrict__ in,
                                                          const float* __restrict__ kerp,
                                                          float* __restrict__ out, const Simt2Params p,
                                                          const __grid_constant__ CUtensorMap tmap_in) {
    // TMA layout: stage buffers 128-B aligned (cp.async.bulk.tensor destination)
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t full_bar[kSimt2MaxStages];   // TMA layout: stage landed (tx bytes)
    const int in_stage = p.in_stage;
    const int ker_stage = p.bc * p.R * KS * p.bko;
    const int stage_floats = TMA ? (in_stage + ker_stage + 31) / 32 * 32 : in_stage + ker_stage;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    int kgi = warp % p.kg;
    const int pwi = warp / p.kg;

    int bx = gridDim.y > 1 ? (int)blockIdx.x : (int)blockIdx.x / p.ktiles;
    int kb = gridDim.y > 1 ? (int)blockIdx.y : (int)blockIdx.x - bx * p.ktiles;
    if (TMA && p.solo) {
        // remainder launch (Simt2Params::solo): 4 warps = 4 of the k tile's channels
        const int b = (int)blockIdx.x / p.solo;
        kgi = ((int)blockIdx.x - b * p.solo) * 4 + warp;
        bx = b / p.ktiles;
        kb = b - bx * p.ktiles;
        bx += p.tile0;
    }
    const int k0 = kb * p.bko;
    const int q = pwi * 32 + lane;
    // n0 / h0: the In box origin (image, row); n_out / h_out: this thread's output row
    int n0, h0, n_out, h_out, g, off;
    bool valid;
    if (p.flat) {
        // flat row mode: slot s0 + q of the flattened (image, row) batch;
        // the box holds the images from the slot tile's first one on
        const int s0 = bx * p.slots;
        n0 = s0 / p.H;
        h0 = 0;
        const int slot = s0 + q;
        n_out = slot / p.H;
        h_out = slot - n_out * p.H;
        g = 0;
        valid = n_out < p.N;
        off = valid ? (n_out - n0) * p.istride + h_out * p.pitch : 0;
    } else {
        const int nt = bx / p.n_htiles;
        const int ht = bx - nt * p.n_htiles;
        n0 = nt * p.tn;
        h0 = ht * p.th;
        // this thread's pixel group: (img, row, g) -> pixels w0 .. w0+TW-1 of one row
        const int per_img = p.th * p.groups;
        const int img = q / p.lpi;
        const int rem = q - img * p.lpi;
        // a padding slot (TMA layout: rem >= per_img) reads the last real slot's
        // window -- the same addresses, a broadcast -- instead of row 0's, which
        // shared 16-B bank groups with the quarter-warp's real rows (ncu r02b:
        // 6 wavefronts per window LDS.128 instead of 4)
        const int remc = rem < per_img ? rem : per_img - 1;
        const int row = remc / p.groups;
        g = remc - row * p.groups;
        valid = q < p.slots && rem < per_img && (n0 + img) < p.N && (h0 + row) < p.H;
        off = q < p.slots ? img * p.istride + row * p.pitch + g * TW : 0;
        n_out = n0 + img;
        h_out = h0 + row;
    }
    const int w0 = g * TW;

#if CONV_SIMT_FFMA2
    // FFMA2 (fma.rn.f32x2, sm_100): output channels in pairs, acc2[i][j] =
    // (acc[2i][j], acc[2i+1][j]) in one 64-bit register pair; each
    // instruction does two FMAs (kernel pair x broadcast input value), so the
    // FMA pipe stays busy with half the issue slots (ncu r02: the FFMA form
    // was issue-bound -- 85 % FFMA, 15 % addressing/LDS, 83 % issue slots busy)
    // (TK = 1, the remainder launch's instance: plain fmaf on acc1)
    unsigned long long acc2[TK / 2 > 0 ? TK / 2 : 1][TW];
    float acc1[TW];
#pragma unroll
    for (int i = 0; i < TK / 2; ++i)
#pragma unroll
        for (int j = 0; j < TW; ++j) acc2[i][j] = 0ull;
#pragma unroll
    for (int j = 0; j < TW; ++j) acc1[j] = 0.0f;
#else
    float acc[TK][TW];
#pragma unroll
    for (int i = 0; i < TK; ++i)
#pragma unroll
        for (int j = 0; j < TW; ++j) acc[i][j] = 0.0f;
#endif

    // Copy plan of the In tile, computed once: a unit is 16 B (4 floats) of
    // one input row when Win % 4 == 0 (rows are then 16-B aligned in NCHW and
    // in smem), else 4 B.  Each thread owns up to kSlots units; per chunk the
    // source only advances by bc channel planes.  Falls back to a row loop
    // when the tile has more units than kSlots * threads.
    constexpr int kSlots = 4;
    const int nrows = p.bc * p.tn * p.rows_in;
    const int upr = p.vec4 ? p.Win / 4 : p.Win;           // units per row
    const int units = nrows * upr;
    const bool slotted = !TMA && units <= kSlots * (int)blockDim.x;
    const int rows_ok = p.Hin - h0 < p.rows_in ? p.Hin - h0 : p.rows_in;
    int64_t s_src[kSlots];
    int s_dst[kSlots], s_cc[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
        const int u = threadIdx.x + k * blockDim.x;
        s_cc[k] = -1; s_dst[k] = 0; s_src[k] = 0;
        if (slotted && u < units) {
            const int rr = u / upr, col = (u - rr * upr) * (p.vec4 ? 4 : 1);
            const int ir = rr % p.rows_in, t2 = rr / p.rows_in;
            const int im = t2 % p.tn, cc = t2 / p.tn;
            const int n = n0 + im;
            s_dst[k] = cc * p.cstride + im * p.istride + ir * p.pitch + col;
            if (n < p.N && ir < rows_ok) {
                s_cc[k] = cc;
                s_src[k] = (((int64_t)n * p.C + cc) * p.Hin + h0 + ir) * p.Win + col;
            } else {
                s_cc[k] = -2;                              // zero-fill
            }
        }
    }
    auto load_stage = [&](int buf, int chunk) {
        float* in_s = sm + buf * stage_floats;
        float* ker_s = in_s + in_stage;
        const int c0 = chunk * p.bc;
        if (slotted) {
            const int64_t adv = (int64_t)c0 * p.Hin * p.Win;
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
                if (s_cc[k] == -1) continue;
                const bool ok = s_cc[k] >= 0 && c0 + s_cc[k] < p.C;
                const float* src = ok ? in + s_src[k] + adv : in;
                if (p.vec4) cp_async16(in_s + s_dst[k], src, ok);
                else cp_async4(in_s + s_dst[k], src, ok);
            }
        } else {
            const int nwarps = blockDim.x >> 5;
            for (int rr = warp; rr < nrows; rr += nwarps) {            // one warp per input row
                const int ir = rr % p.rows_in;
                const int t2 = rr / p.rows_in;
                const int im = t2 % p.tn;
                const int cc = t2 / p.tn;
                const int c = c0 + cc, n = n0 + im;
                const bool ok = c < p.C && n < p.N && ir < rows_ok;
                const float* src = in + (((int64_t)n * p.C + c) * p.Hin + h0 + ir) * p.Win;
                float* dst = in_s + cc * p.cstride + im * p.istride + ir * p.pitch;
                if (p.vec4)      // 16-B aligned rows (same addressing as the slotted plan)
                    for (int col = lane * 4; col < p.Win; col += 128) cp_async16(dst + col, ok ? src + col : in, ok);
                else
                    for (int col = lane; col < p.Win; col += 32) cp_async4(dst + col, ok ? src + col : in, ok);
            }
        }
        // Ker: contiguous slab of the packed tensor, channels >= C zero.
        const int cvalid = p.C - c0 < p.bc ? p.C - c0 : p.bc;
        const int len_ok = cvalid * p.R * KS * p.bko;
        const float* gk = kerp + (((int64_t)kb * p.C + c0) * p.R * KS) * p.bko;
        for (int e = threadIdx.x * 4; e < ker_stage; e += blockDim.x * 4)
            cp_async16(ker_s + e, e < len_ok ? gk + e : kerp, e < len_ok);
    };

    // TMA layout: one 4-D box {pitch columns, rows_in rows, bc channels, tn
    // images} of In (columns >= Win, rows >= Hin, channels >= C and images
    // >= N zero-filled) plus one bulk copy of the packed Ker slab, issued by
    // one thread and completing on the stage's mbarrier (ncu r02: the
    // per-thread cp.async plan cost ~300 issue slots per warp per chunk,
    // ~8 % of the kernel's instructions)
    auto issue_stage = [&](int buf, int chunk) {
        float* in_s = sm + buf * stage_floats;
        float* ker_s = in_s + in_stage;
        const int c0 = chunk * p.bc;
        const int cvalid = p.C - c0 < p.bc ? p.C - c0 : p.bc;
        const uint32_t kbytes = (uint32_t)cvalid * p.R * KS * p.bko * 4u;
        sm100::mbar_arrive_expect_tx(&full_bar[buf], p.tx_in + kbytes);
        if (p.flat) sm100::tma_load_4d(in_s, &tmap_in, &full_bar[buf], 0, 0, n0, c0);   // dims {Win, Hin, N, C}
        else sm100::tma_load_4d(in_s, &tmap_in, &full_bar[buf], 0, h0, c0, n0);
        sm100::bulk_load_g2s(ker_s, kerp + (((int64_t)kb * p.C + c0) * p.R * KS) * p.bko, kbytes, &full_bar[buf]);
    };

    constexpr int WIN = TW + KS - 1;
    constexpr int WIN4 = (WIN + 3) / 4 * 4;
    // warp-shuffle halo (north_star's wording): pixel-group mode TW = 4,
    // S = 3 only -- in row mode a lane's window is its whole input row and
    // no neighbour holds any of it.  r02b A/B over the 19 Table-1 layers
    // that take TW = 4 (profiles/r02b/simt_shfl_ab/): TK = 8 tiles 0.77-1.00x
    // (Y0 -23 %, M5 -4 %, none slower than +0.4 %), TK = 4 tiles up to 6 %
    // slower (Y2, Y8) -- so the shuffle halo is compiled for TK = 8 only
    constexpr bool kShflHalo = TW == 4 && KS == 3 && (CONV_SIMT_SHFL == 1 || (CONV_SIMT_SHFL == 2 && TK == 8));
    const bool own_halo = g == p.groups - 1 || lane == 31;
    if (!(TMA && p.nowait)) asm volatile("griddepcontrol.wait;" ::: "memory");   // packed Ker written by the previous grid
    if (TMA && p.trigger) asm volatile("griddepcontrol.launch_dependents;");     // the other grid may start (Ker complete)
    // split-C (separate instances, so the plain loop keeps its exact code --
    // the runtime range measured 3.5 % slower on the batched layer): this
    // CTA's channel chunks [c_beg, c_end) and its partial-output slab
    const int c_beg = SPLITC ? (int)blockIdx.z * p.cper : 0;
    const int c_end = SPLITC ? min(p.nchunks, c_beg + p.cper) : p.nchunks;
    if (SPLITC) out += (int64_t)blockIdx.z * p.zstride;
    // three-stage ring, one barrier per chunk: the copies of chunk i+2 are
    // issued after the barrier that ends every thread's use of chunk i-1's
    // buffer (ncu r02: with two stages and two barriers per chunk a third of
    // the stall samples sat outside the FFMA loop, in the waits)
    // (TMA layout: p.stages deep, chunk i + stages - 1 issued into chunk
    // i-1's buffer after the barrier)
    const int S = TMA ? p.stages : kSimt2Stages;
    if (TMA) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < S; ++i) sm100::mbar_init(&full_bar[i], 1);
            sm100::fence_barrier_init();
            for (int i = 0; i < S - 1 && c_beg + i < c_end; ++i) issue_stage(i, c_beg + i);
        }
    } else {
        load_stage(0, c_beg);
        cp_async_commit();
        if (c_beg + 1 < c_end) load_stage(1, c_beg + 1);
        cp_async_commit();
    }
    int buf = 0;
    uint32_t phase = 0;
    for (int chunk = c_beg; chunk < c_end; ++chunk) {
        const int ci = chunk - c_beg;
        if (TMA) {
            __syncthreads();                      // every thread is done with chunk i-1's buffer
            if (threadIdx.x == 0 && chunk + S - 1 < c_end) issue_stage(buf == 0 ? S - 1 : buf - 1, chunk + S - 1);
            sm100::mbar_wait(&full_bar[buf], phase);
        } else {
            cp_async_wait<1>();                   // chunk i has landed (i+1 may be in flight)
            __syncthreads();
            if (chunk + 2 < c_end) load_stage((ci + 2) % kSimt2Stages, chunk + 2);
            cp_async_commit();
        }
        const float* in_s = sm + buf * stage_floats;
        const float* ker_s = in_s + in_stage;
        const int cc_end = p.C - chunk * p.bc < p.bc ? p.C - chunk * p.bc : p.bc;
        const int R = KR ? KR : p.R;
        // row mode unrolls the channel loop by 2 so that the next channel's
        // window and kernel loads overlap this one's FFMA2s (r02b: batched
        // 1199 -> 1190 us; for the TW = 4 / 8 instances it lost 3 % on
        // Table 1, Y0 +35 %: profiles/r02b/simt_cc_unroll_ab/)
        constexpr int kCcUnroll = CONV_SIMT_CC_UNROLL > 0 ? CONV_SIMT_CC_UNROLL : (TW >= 7 ? 2 : 1);
#pragma unroll kCcUnroll
        for (int cc = 0; cc < cc_end; ++cc) {
            const float* ip = in_s + cc * p.cstride + off;
            const float* kp = ker_s + cc * R * KS * p.bko + kgi * TK;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float win[WIN4];
                if (kShflHalo) {
                    // north_star's warp-shuffle reuse (A/B build): the lane's
                    // own 4 inputs by one LDS.128, the 2-float halo from the
                    // next lane (the next pixel group of the row), or by an
                    // LDS.64 where that lane is in another row or warp
                    const float4 v = *reinterpret_cast<const float4*>(ip + r * p.pitch);
                    win[0] = v.x; win[1] = v.y; win[2] = v.z; win[3] = v.w;
                    float h0 = __shfl_down_sync(0xffffffffu, v.x, 1);
                    float h1 = __shfl_down_sync(0xffffffffu, v.y, 1);
                    if (own_halo) {
                        const float2 t = *reinterpret_cast<const float2*>(ip + r * p.pitch + 4);
                        h0 = t.x; h1 = t.y;
                    }
                    win[4] = h0; win[5] = h1;
                } else {
#pragma unroll
                    for (int j = 0; j < WIN4; j += 4) {
                        const float4 v = *reinterpret_cast<const float4*>(ip + r * p.pitch + j);
                        win[j] = v.x; win[j + 1] = v.y; win[j + 2] = v.z; win[j + 3] = v.w;
                    }
                }
#pragma unroll
                for (int s = 0; s < KS; ++s) {
#if CONV_SIMT_FFMA2
                    if constexpr (TK == 1) {
                        const float kv1 = kp[(r * KS + s) * p.bko];
#pragma unroll
                        for (int j = 0; j < TW; ++j) acc1[j] = fmaf(kv1, win[j + s], acc1[j]);
                    } else {
                    unsigned long long kv2[TK / 2 > 0 ? TK / 2 : 1];
#pragma unroll
                    for (int i = 0; i + 3 < TK; i += 4) {
                        const float4 k4 = *reinterpret_cast<const float4*>(kp + (r * KS + s) * p.bko + i);
                        asm("mov.b64 %0, {%1, %2};" : "=l"(kv2[i / 2]) : "f"(k4.x), "f"(k4.y));
                        asm("mov.b64 %0, {%1, %2};" : "=l"(kv2[i / 2 + 1]) : "f"(k4.z), "f"(k4.w));
                    }
#pragma unroll
                    for (int j = 0; j < TW; ++j) {
                        unsigned long long w2;
                        asm("mov.b64 %0, {%1, %1};" : "=l"(w2) : "f"(win[j + s]));   // folds into a .F32 operand
#pragma unroll
                        for (int i = 0; i < TK / 2; ++i)
                            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[i][j]) : "l"(kv2[i]), "l"(w2));
                    }
                    }
#else
                    float kv[TK];
                    if constexpr (TK == 1) kv[0] = kp[(r * KS + s) * p.bko];
#pragma unroll
                    for (int i = 0; i + 3 < TK; i += 4) {
                        const float4 k4 = *reinterpret_cast<const float4*>(kp + (r * KS + s) * p.bko + i);
                        kv[i] = k4.x; kv[i + 1] = k4.y; kv[i + 2] = k4.z; kv[i + 3] = k4.w;
                    }
                    // (pixel-outer order, to pair accumulators and kernel
                    // values in opposite register banks: ptxas reorders it
                    // anyway and the layer ran 3.6 % slower, r02b)
#pragma unroll
                    for (int i = 0; i < TK; ++i)
#pragma unroll
                        for (int j = 0; j < TW; ++j) acc[i][j] = fmaf(kv[i], win[j + s], acc[i][j]);
#endif
                }
            }
        }
        if (++buf == S) { buf = 0; phase ^= 1u; }
    }

    if (TMA && p.endwait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!valid) return;
#if CONV_SIMT_FFMA2
    float acc[TK][TW];
#pragma unroll
    for (int i = 0; i < TK / 2; ++i)
#pragma unroll
        for (int j = 0; j < TW; ++j) {
            acc[2 * i][j] = __uint_as_float((uint32_t)acc2[i][j]);
            acc[2 * i + 1][j] = __uint_as_float((uint32_t)(acc2[i][j] >> 32));
        }
    if constexpr (TK == 1) {
#pragma unroll
        for (int j = 0; j < TW; ++j) acc[0][j] = acc1[j];
    }
#endif
#pragma unroll
    for (int i = 0; i < TK; ++i) {
        const int k = k0 + kgi * TK + i;
        if (k >= p.K) break;
        float* o = out + (((int64_t)n_out * p.K + k) * p.H + h_out) * p.W + w0;
#pragma unroll
        for (int j = 0; j < TW; ++j)
            if (w0 + j < p.W) o[j] = acc[i][j];
    }
}

bool simt_tile_supported(const SimtTile& t) {
    if (t.tk != 4 && t.tk != 8) return false;
    if (t.tw < 1 || t.tw > 14) return false;
    if (t.ver != 2 && t.tw > 8) return false;
    // v2: 4 / 8 pixels per thread (16-B aligned windows), or a whole output
    // row of 7 or 14 pixels (row mode, TK = 4: 56 accumulators)
    // (row mode with TK = 8 -- 112 accumulators, 254 registers, one 256-thread
    // CTA per SM -- measured 13 % slower on the batched layer, r02
    // profiles/r02/simt_sweep_tk8.jsonl; not instantiated)
    if (t.ver == 2 && t.tw != 4 && t.tw != 8 && !((t.tw == 7 || t.tw == 14) && t.tk == 4)) return false;
    const int threads = 32 * t.kg * t.pw;
    const int max_threads = (t.ver == 2 && t.tk * t.tw > 64) ? 256 : 512;   // Simt2Threads
    return t.kg >= 1 && t.pw >= 1 && threads <= max_threads && t.tn >= 1 && t.th >= 1 && t.bc >= 1;
}

bool simt_v2_ok(const Problem& pb) { return pb.U == 1 && pb.D == 1 && pb.ph == 0 && pb.pw == 0 && (pb.S == 1 || pb.S == 3); }

// Row mode (TW = 7 or 14): one thread per output row, allowed only when the
// row is exactly that wide (its window then starts 16-B aligned at w = 0).
bool simt_v2_tw_ok(const Problem& pb, int tw) { return tw == 4 || tw == 8 || tw == pb.W; }

// v2 smem row pitch: the last group's window (WIN rounded up to 4) must fit;
// multiple of 4 floats; rows of <= 16 floats of groups are offset by 16 mod 32
// floats so that a quarter-warp's 128-bit window loads hit distinct banks.
int simt2_pitch(const Problem& pb, const SimtTile& t) {
    const int groups = (pb.W + t.tw - 1) / t.tw;
    const int win4 = (t.tw + pb.S - 1 + 3) / 4 * 4;
    int pitch = std::max((int)pb.Win(), (groups - 1) * t.tw + win4);
    pitch = (pitch + 3) / 4 * 4;
    if (groups == 1) {
        // row mode: consecutive lanes are consecutive rows; an odd number of
        // 16-B units per row puts a quarter-warp's 8 window loads on 8
        // distinct 16-B bank groups
        if ((pitch / 4) % 2 == 0) pitch += 4;
    } else if (pitch % 32 == 0) {
        pitch += 4;                       // rows 128 B apart would put every row's window on the same banks
    }
    return pitch;
}

// v2 image stride in smem: row mode with few rows per image (th < 8) puts
// several images in one quarter-warp; their windows are then 16-B units
// i*istride/4 + r*pitch/4 apart, and an image stride of 2 or 6 (mod 8) units
// with the odd pitch keeps the 8 loads on distinct bank groups (without it
// the lane-filling tn = 16, th = 2 tile ran 2-way conflicted, r02)
int simt2_istride(const Problem& pb, const SimtTile& t) {
    const int pitch = simt2_pitch(pb, t);
    int units = (int)pb.rows_span(t.th) * pitch / 4;
    const bool row_mode = (pb.W + t.tw - 1) / t.tw == 1;
    if (row_mode && t.th < 8)
        while (units % 8 != 2 && units % 8 != 6) ++units;
    return units * 4;
}

// v2 shared-memory layout of one stage.  The TMA layout is taken when In
// rows are 16-B multiples (Win % 4 == 0, the TMA stride rule), the box fits
// TMA's 256-element dims, R is a compiled tap count, and each image's slots
// can be padded to whole quarter-warps: the box lands dense as
// [img][c][row][pitch], so the image stride (bc * rows * pitch) is not free
// to choose, and a quarter-warp that straddled two images could conflict.
// CONV_SIMT_NO_TMA=1 keeps the per-thread cp.async layout, CONV_SIMT_STAGES=n
// sets the TMA ring depth (2..4; A/B).
Simt2Layout simt2_layout(const Problem& pb, const SimtTile& t) {
    Simt2Layout L;
    L.pitch = simt2_pitch(pb, t);
    const int rows_in = (int)pb.rows_span(t.th);
    const int groups = (pb.W + t.tw - 1) / t.tw;
    const int per_img = t.th * groups;
    const int lpi8 = (per_img + 7) / 8 * 8;
    static const bool no_tma = getenv("CONV_SIMT_NO_TMA") != nullptr;
    static const int env_stages = getenv("CONV_SIMT_STAGES") ? atoi(getenv("CONV_SIMT_STAGES")) : 0;
    L.tma = !no_tma && t.ver == 2 && simt_v2_ok(pb) && pb.Win() % 4 == 0 && L.pitch <= 256 && rows_in <= 256 &&
            t.bc <= 256 && t.tn <= 256 && pb.R == pb.S && (pb.S == 1 || pb.S == 3) &&   // the compiled TMA instances
            (t.flat || t.tn * lpi8 <= 32 * t.pw);                                       // (dispatch_simt2): 1x1 and 3x3 taps
    // (r02e fuzz: the test was R in {1, 3}, which let 1x3 problems with Win % 4 == 0 plan a TMA tile that no
    // instance runs -- the launch failed with invalid argument; they take the cp.async layout now)
    // (flat tiles: a 2-deep ring by default -- their boxes carry the zero
    // rows up to rows_box, and 3 stages would cost a resident CTA per SM)
    L.stages = L.tma && env_stages >= 2 && env_stages <= kSimt2MaxStages ? env_stages : t.flat ? 2 : kSimt2Stages;
    const int ker_stage = t.bc * pb.R * pb.S * t.kg * t.tk;
    if (t.flat) {
        // flat row mode: smem [c][img][rows_box][pitch] (the tensor map's
        // image and channel dims swapped), rows_box = rows_in rounded up to
        // = H (mod 8).  Slot q of the CTA sits at (img*rows_box + row)*pitch;
        // with an odd number of 16-B units per row, 8 consecutive slots then
        // fall on 8 distinct bank groups even where they cross an image
        // (img*rows_box + row = q + img*(rows_box - H)).
        const bool ok = L.tma && groups == 1 && t.th == pb.H;
        L.tma = ok;
        if (!ok) { L.in_stage = -1; return L; }
        int rb = rows_in;
        while ((rb - pb.H) % 8 != 0) ++rb;
        L.rows_box = rb;
        const int nb = simt_flat_images(pb, t);
        if (rb > 256 || nb > 256) { L.tma = false; L.in_stage = -1; return L; }
        L.istride = rb * L.pitch;
        L.cstride = nb * L.istride;
        L.in_stage = t.bc * L.cstride;
        L.lpi = pb.H;
        L.stage_floats = (L.in_stage + ker_stage + 31) / 32 * 32;
    } else if (L.tma) {
        L.rows_box = rows_in;
        L.cstride = rows_in * L.pitch;
        L.istride = t.bc * L.cstride;            // the box is dense: [img][c][row][pitch]
        L.in_stage = t.tn * L.istride;
        L.lpi = lpi8;
        L.stage_floats = (L.in_stage + ker_stage + 31) / 32 * 32;
    } else {
        L.istride = simt2_istride(pb, t);
        L.cstride = t.tn * L.istride;
        L.in_stage = t.bc * L.cstride;
        L.lpi = per_img;
        L.stage_floats = L.in_stage + ker_stage;
    }
    return L;
}

// Remainder launch of a flat tile (internal.h).  The kernel's time goes with
// the CTAs per SM, k = ceil(CTAs / SMs) (T = 35 + 87 k us on the batched
// layer); when (k - 1) * SMs CTAs hold all but `rem` slot tiles, those run
// as rem * ktiles * kg one-warp CTAs -- at most one per SM, and small enough
// (2-channel chunks) to fit beside the main grid's resident CTAs -- so the
// busiest SM carries k - 1 CTAs and one warp instead of k CTAs (r02d,
// batched layer: 1792 CTAs = 12.1 per SM -> 1776 + 64 warps).
SimtTile simt_rem_tile(const SimtTile& t) {
    SimtTile ts = t;
    ts.bc = std::min(t.bc, 2);
    ts.kg = t.kg * t.tk;      // same k tile (bko channels) and packed Ker, one channel per k group
    ts.tk = 1;
    return ts;
}

int simt_rem_tiles(const Problem& pb, const SimtTile& t, int sms) {
    static const bool off = getenv("CONV_SIMT_NO_REM") != nullptr;   // A/B
    if (off || !t.flat || !t.rem || t.ver != 2 || t.pw != 1 || t.kg < 2 || sms < 1) return 0;
    // the remainder instance is compiled for 3x3 taps and 14-pixel rows only (dispatch_simt2); other flat
    // problems (W = 14, S = 3, R != 3) run the main grid alone (r02e fuzz: the launch failed with R = 1, 2, 5)
    if (pb.R != 3 || pb.S != 3 || t.tw != 14 || t.tk != 4) return 0;
    // split-C (r02e): a slot tile is k tiles x splits CTAs; the remainder grid takes the same
    // channel ranges in its own 2-channel chunks (needs an even chunk depth) and writes the
    // same partial slabs
    const int64_t nchunks = (pb.C + t.bc - 1) / t.bc;
    const int64_t splits = std::max<int64_t>(1, std::min<int64_t>(t.splits, nchunks));
    const int64_t cper = (nchunks + splits - 1) / splits;
    const int64_t zsplits = (nchunks + cper - 1) / cper;
    if (zsplits > 1 && t.bc % 2 != 0) return 0;
    const int64_t ktiles = (pb.K + (int64_t)t.kg * t.tk - 1) / ((int64_t)t.kg * t.tk) * zsplits;
    const int64_t tiles = ((int64_t)pb.N * pb.H + 31) / 32;           // slot tiles (pw = 1)
    const int64_t ctas = tiles * ktiles;
    const int64_t k = (ctas + sms - 1) / sms;
    if (k < 2) return 0;
    const int64_t main_tiles = (k - 1) * sms / ktiles;
    const int64_t rem = tiles - main_tiles;
    if (rem < 1 || main_tiles < 1 || rem * ktiles * (t.kg * t.tk / 4) > sms) return 0;
    // shared memory: the main grid's resident CTAs + one remainder CTA per SM
    const SimtTile ts = simt_rem_tile(t);
    const size_t sm_main = simt_smem_bytes(pb, t), sm_rem = simt_smem_bytes(pb, ts);
    if (sm_main == SIZE_MAX || sm_rem == SIZE_MAX || !simt2_layout(pb, ts).tma) return 0;
    const int64_t threads = 32 * t.kg;
    const int64_t per_sm = std::min<int64_t>({(int64_t)(228 * 1024 / (sm_main + 1024)), (2048 - 128) / threads,
                                              (65536 - 64 * 128) / (128 * threads), k - 1});
    if (per_sm < 1 || per_sm * (sm_main + 1024) + (sm_rem + 1024) > (size_t)228 * 1024) return 0;
    return (int)rem;
}

size_t simt_smem_bytes(const Problem& pb, const SimtTile& t) {
    if (t.ver == 2) {
        const Simt2Layout L = simt2_layout(pb, t);
        if (L.in_stage < 0) return SIZE_MAX;      // infeasible (flat without the TMA layout)
        // TMA layout: + the mbarriers' 128-B aligned static slot
        return (size_t)L.stages * L.stage_floats * sizeof(float) + (L.tma ? 128 : 0);
    }
    const size_t row = (size_t)(pb.Win() + 2 * pb.pw);
    const size_t plane = (size_t)t.tn * pb.rows_span(t.th) * row;
    const size_t in_stage = (size_t)t.bc * plane;
    const size_t ker_stage = (size_t)t.bc * pb.R * pb.S * t.kg * t.tk;
    return 2 * (in_stage + ker_stage) * sizeof(float);
}

// Launch one SIMT kernel instance, opting it in to the largest dynamic smem
// per device (`smem_set` is that instance's own flags).
template <typename K, typename P>
static cudaError_t launch_simt_inst(K kfn, SmemOptIn& smem_set, const float* in, const float* kerp, float* out,
                                    const P& p, dim3 grid, int threads, size_t smem, cudaStream_t st) {
    if (cudaError_t e = smem_set.ensure(kfn, smem); e != cudaSuccess) return e;
    return launch_pdl(kfn, grid, threads, smem, st, in, kerp, out, p);
}

template <int TK, int TW, int KR, int KS, bool TMA>
static cudaError_t launch_simt2_t(const float* in, const float* kerp, float* out, const Simt2Params& p,
                                  const CUtensorMap& tmap, dim3 grid, int threads, size_t smem, cudaStream_t st) {
    static SmemOptIn set_plain, set_split;
    const size_t dyn = TMA ? smem - 128 : smem;
    if (grid.z > 1) {
        auto kfn = conv_direct_simt2<TK, TW, KR, KS, true, TMA>;
        if (cudaError_t e = set_split.ensure(kfn, dyn); e != cudaSuccess) return e;
        return launch_pdl(kfn, grid, threads, dyn, st, in, kerp, out, p, tmap);
    }
    auto kfn = conv_direct_simt2<TK, TW, KR, KS, false, TMA>;
    if (cudaError_t e = set_plain.ensure(kfn, dyn); e != cudaSuccess) return e;
    return launch_pdl(kfn, grid, threads, dyn, st, in, kerp, out, p, tmap);
}


static cudaError_t dispatch_simt2(const SimtTile& t, int R, int S, bool tma, const float* in, const float* kerp,
                                  float* out, const Simt2Params& p, const CUtensorMap& tmap, dim3 grid, int threads,
                                  size_t smem, cudaStream_t st) {
    // TMA instances only for the compiled tap counts (R = S in {1, 3})
#define SIMT2_CASE(TK_, TW_, R_, S_) \
    if (t.tk == TK_ && t.tw == TW_ && (R_ == 0 || R == R_) && S == S_) { \
        if (R_ != 0 && tma) return launch_simt2_t<TK_, TW_, R_, S_, (R_ != 0)>(in, kerp, out, p, tmap, grid, threads, smem, st); \
        if (!tma) return launch_simt2_t<TK_, TW_, R_, S_, false>(in, kerp, out, p, tmap, grid, threads, smem, st); \
    }
    SIMT2_CASE(4, 4, 1, 1) SIMT2_CASE(4, 8, 1, 1) SIMT2_CASE(8, 4, 1, 1) SIMT2_CASE(8, 8, 1, 1)
    SIMT2_CASE(4, 4, 3, 3) SIMT2_CASE(4, 8, 3, 3) SIMT2_CASE(8, 4, 3, 3) SIMT2_CASE(8, 8, 3, 3)
    SIMT2_CASE(4, 4, 0, 1) SIMT2_CASE(4, 8, 0, 1) SIMT2_CASE(8, 4, 0, 1) SIMT2_CASE(8, 8, 0, 1)
    SIMT2_CASE(4, 4, 0, 3) SIMT2_CASE(4, 8, 0, 3) SIMT2_CASE(8, 4, 0, 3) SIMT2_CASE(8, 8, 0, 3)
    SIMT2_CASE(4, 14, 3, 3) SIMT2_CASE(4, 7, 3, 3) SIMT2_CASE(4, 14, 1, 1) SIMT2_CASE(4, 7, 1, 1)
    SIMT2_CASE(4, 14, 0, 3) SIMT2_CASE(4, 7, 0, 3) SIMT2_CASE(4, 14, 0, 1) SIMT2_CASE(4, 7, 0, 1)
    // the remainder launch's instance (simt_rem_tile: flat tiles exist for W = 14, R = S = 3 only)
    if (t.tk == 1 && t.tw == 14 && R == 3 && S == 3 && tma)
        return launch_simt2_t<1, 14, 3, 3, true>(in, kerp, out, p, tmap, grid, threads, smem, st);
#undef SIMT2_CASE
    return cudaErrorInvalidValue;
}

template <int TK, int TW>
static cudaError_t launch_simt_t(const float* in, const float* kerp, float* out, const SimtParams& p,
                                 dim3 grid, int threads, size_t smem, cudaStream_t st) {
    static SmemOptIn set_plain, set_split;
    if (grid.z > 1)
        return launch_simt_inst(conv_direct_simt<TK, TW, true>, set_split, in, kerp, out, p, grid, threads, smem, st);
    return launch_simt_inst(conv_direct_simt<TK, TW, false>, set_plain, in, kerp, out, p, grid, threads, smem, st);
}


#define SIMT_CASE(TK_, TW_) \
    if (t.tk == TK_ && t.tw == TW_) return launch_simt_t<TK_, TW_>(in, kerp, out, p, grid, threads, smem, st);

static cudaError_t dispatch_simt(const SimtTile& t, const float* in, const float* kerp, float* out,
                                 const SimtParams& p, dim3 grid, int threads, size_t smem, cudaStream_t st) {
    SIMT_CASE(4, 1) SIMT_CASE(4, 2) SIMT_CASE(4, 3) SIMT_CASE(4, 4)
    SIMT_CASE(4, 5) SIMT_CASE(4, 6) SIMT_CASE(4, 7) SIMT_CASE(4, 8)
    SIMT_CASE(8, 1) SIMT_CASE(8, 2) SIMT_CASE(8, 3) SIMT_CASE(8, 4)
    SIMT_CASE(8, 5) SIMT_CASE(8, 6) SIMT_CASE(8, 7) SIMT_CASE(8, 8)
    return cudaErrorInvalidValue;
}

static size_t simt_pack_bytes(const Problem& pb, const SimtTile& t) {
    const int bko = t.kg * t.tk;
    const size_t kb = (size_t)(pb.K + bko - 1) / bko;
    return (kb * bko * (size_t)pb.C * pb.R * pb.S * sizeof(float) + 255) / 256 * 256;
}

size_t simt_ws_bytes(const Problem& pb, const SimtTile& t) {
    const size_t part = t.splits > 1 ? (size_t)t.splits * pb.out_elems() * sizeof(float) : 0;
    return simt_pack_bytes(pb, t) + part;
}

cudaError_t simt_run(const Problem& pb, const SimtTile& t, const float* in, const float* ker,
                     float* out, void* ws, cudaStream_t st, cudaEvent_t* ev, std::string& err, int sms, bool skip_pack) {
    SimtParams p;
    p.N = pb.N; p.K = pb.K; p.C = pb.C; p.H = pb.H; p.W = pb.W; p.R = pb.R; p.S = pb.S; p.U = pb.U; p.D = pb.D;
    p.Hin = (int)pb.Hin(); p.Win = (int)pb.Win(); p.HW = pb.H * pb.W; p.RS = pb.R * pb.S;
    p.tn = t.tn; p.th = t.th; p.bc = t.bc; p.kg = t.kg;
    p.bko = t.kg * t.tk;
    p.rows_in = (int)pb.rows_span(t.th);
    p.ph = pb.ph;
    p.pw = pb.pw;
    p.pitch = p.Win + 2 * pb.pw;
    p.plane = t.tn * p.rows_in * p.pitch;
    p.n_htiles = (pb.H + t.th - 1) / t.th;
    p.nchunks = (pb.C + t.bc - 1) / t.bc;
    const int splits = std::max(1, std::min(t.splits, p.nchunks));
    p.cper = (p.nchunks + splits - 1) / splits;
    const int zsplits = (p.nchunks + p.cper - 1) / p.cper;     // non-empty splits
    p.zstride = zsplits > 1 ? pb.out_elems() : 0;
    float* kout = zsplits > 1 ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + simt_pack_bytes(pb, t)) : out;
    p.bp = t.tn * t.th * pb.W;
    p.vec4_in = (p.Win % 4 == 0) ? 1 : 0;
    if (t.ver != 2 && p.bp > t.pw * 32 * t.tw) { err = "SIMT tile: pixel slots < tn*th*W"; return cudaErrorInvalidValue; }
    if (t.ver == 2 && !simt_v2_ok(pb)) { err = "SIMT v2 needs stride 1, dilation 1, no padding, S in {1, 3}"; return cudaErrorInvalidValue; }

    float* kerp = static_cast<float*>(ws);
    const int64_t total = (int64_t)((pb.K + p.bko - 1) / p.bko) * p.bko * pb.C * p.RS;
    const int pblocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    if (ev) cudaEventRecord(ev[0], st);
    // the tiled transpose, except for small packs with C*R*S % 4 != 0 (its
    // scalar form measured r02c, profiles/r02c/pack/: Y0 8.4 vs 7.1 us, R1
    // 8.7 vs 6.9 for the gather; with 16-B units it is at least as fast on
    // every Table-1 layer, M9 66.8 -> 21.2 us, Y23 183 -> 55, batched 12.3 ->
    // 8.0)
    static const int gather_env = getenv("CONV_SIMT_PACK_GATHER") ? atoi(getenv("CONV_SIMT_PACK_GATHER")) : -1;
    const bool gather = gather_env == 1 ||
                        (gather_env != 0 && (pb.C * p.RS) % 4 != 0 && total < (int64_t)1 << 18);
    // skip_pack (conv_run_host's later chunks): the workspace already holds this tile's packed Ker
    if (skip_pack) {
    } else if (gather || p.bko > 1024) {
        pack_ker_simt<<<pblocks, 256, 0, st>>>(ker, kerp, pb.K, pb.C, p.RS, p.bko, total);
    } else {
        const int crs = pb.C * p.RS;
        const int cw = 1024 / p.bko;                         // bko is a multiple of 4 up to 64
        const int nchunk = (crs + cw - 1) / cw;
        const int64_t nblk = (int64_t)((pb.K + p.bko - 1) / p.bko) * nchunk;
        pack_ker_simt_tiled<<<(unsigned)nblk, 256, 0, st>>>(ker, kerp, pb.K, crs, p.bko, cw, nchunk);
    }
    if (ev) cudaEventRecord(ev[1], st);

    const int n_ntiles = (pb.N + t.tn - 1) / t.tn;
    dim3 grid((unsigned)(n_ntiles * p.n_htiles), (unsigned)((pb.K + p.bko - 1) / p.bko), (unsigned)zsplits);
    const int threads = 32 * t.kg * t.pw;
    const size_t smem = simt_smem_bytes(pb, t);
    cudaError_t e;
    if (t.ver == 2) {
        Simt2Params q;
        q.N = pb.N; q.K = pb.K; q.C = pb.C; q.H = pb.H; q.W = pb.W; q.R = pb.R; q.S = pb.S;
        q.Hin = (int)pb.Hin(); q.Win = (int)pb.Win();
        q.tn = t.tn; q.th = t.th; q.bc = t.bc; q.kg = t.kg; q.bko = p.bko;
        q.rows_in = p.rows_in;
        const Simt2Layout L = simt2_layout(pb, t);
        q.pitch = L.pitch;
        q.istride = L.istride;
        q.cstride = L.cstride;
        q.plane = L.cstride;
        q.in_stage = L.in_stage;
        q.lpi = L.lpi;
        q.groups = (pb.W + t.tw - 1) / t.tw;
        q.n_htiles = p.n_htiles;
        q.nchunks = p.nchunks;
        q.cper = p.cper;
        q.zstride = p.zstride;
        q.flat = t.flat ? 1 : 0;
        if (t.flat && !L.tma) { err = "SIMT flat tile needs the TMA row-mode layout (th = H, TW = W, Win % 4 == 0)"; return cudaErrorInvalidValue; }
        const int box_imgs = t.flat ? simt_flat_images(pb, t) : t.tn;
        q.slots = t.flat ? 32 * t.pw : t.tn * L.lpi;
        if (q.slots > t.pw * 32) { err = "SIMT v2 tile: pixel-group slots > pw*32"; return cudaErrorInvalidValue; }
        q.vec4 = (q.Win % 4 == 0) ? 1 : 0;
        q.tx_in = (uint32_t)((size_t)box_imgs * t.bc * L.rows_box * q.pitch * sizeof(float));
        if (t.flat) grid.x = (unsigned)(((int64_t)pb.N * pb.H + q.slots - 1) / q.slots);
        q.stages = L.stages;
        q.ktiles = (pb.K + p.bko - 1) / p.bko;
        static const bool grid2d = getenv("CONV_SIMT_GRID2D") != nullptr;   // A/B: the r02 2-D grid (k tile = y)
        if (!grid2d) grid = dim3(grid.x * grid.y, 1, grid.z);
        else q.ktiles = 1;
        CUtensorMap tmap;
        memset(&tmap, 0, sizeof(tmap));
        // In NCHW as {Win, Hin, C, N}; box {pitch, rows_in, bc, tn}: columns
        // >= Win (the pitch padding), rows >= Hin, channels >= C and
        // images >= N are zero-filled
        // (flat: {Win, Hin, N, C}, box {pitch, rows_box, images, bc} -- the
        // image dim inside the channel dim, so a channel's images are
        // consecutive row blocks in smem)
        auto encode = [&](CUtensorMap* tm, const Simt2Layout& Lx, int bc) -> bool {
            if (!driver_init(err)) return false;
            const cuuint64_t plane_b = (cuuint64_t)q.Hin * q.Win * 4, image_b = (cuuint64_t)pb.C * plane_b;
            cuuint64_t dims[4] = {(cuuint64_t)q.Win, (cuuint64_t)q.Hin, (cuuint64_t)(t.flat ? pb.N : pb.C),
                                  (cuuint64_t)(t.flat ? pb.C : pb.N)};
            cuuint64_t strides[3] = {(cuuint64_t)q.Win * 4, t.flat ? image_b : plane_b, t.flat ? plane_b : image_b};
            cuuint32_t box[4] = {(cuuint32_t)Lx.pitch, (cuuint32_t)Lx.rows_box, (cuuint32_t)(t.flat ? box_imgs : bc),
                                 (cuuint32_t)(t.flat ? bc : t.tn)};
            cuuint32_t estr[4] = {1, 1, 1, 1};
            CUresult r = g_encode_tiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in), dims, strides,
                                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { err = "cuTensorMapEncodeTiled (SIMT In) failed (" + std::to_string((int)r) + ")"; return false; }
            return true;
        };
        if (L.tma && !encode(&tmap, L, t.bc)) return cudaErrorInvalidValue;
        q.solo = 0; q.tile0 = 0; q.nowait = 0; q.trigger = 0; q.endwait = 0;
        // Remainder launch (simt_rem_tiles): the last `rem` slot tiles run as
        // 4-warp CTAs of the TK = 1 instance with 2-channel chunks -- each
        // warp one output channel of the CTA's 4, so the four SMSPs of the SM
        // get a quarter of a main warp's FMAs each -- small enough to sit
        // beside the main grid's resident CTAs.  Launched first; the main
        // grid follows as their programmatic dependent (released once they
        // have seen the packed Ker complete), does not wait for their end
        // before it starts, and waits for it at the end of each CTA, so that
        // the main grid's end implies the remainder grid's.  Per output the
        // arithmetic is the main tile's (same c, r, s order of fmaf).
        const int rem = (L.tma && !grid2d) ? simt_rem_tiles(pb, t, sms) : 0;
        if (rem > 0) {
            const SimtTile ts = simt_rem_tile(t);
            const Simt2Layout Ls = simt2_layout(pb, ts);
            Simt2Params qs = q;
            qs.bc = ts.bc; qs.kg = ts.kg;
            qs.pitch = Ls.pitch; qs.istride = Ls.istride; qs.cstride = Ls.cstride; qs.plane = Ls.cstride;
            qs.in_stage = Ls.in_stage; qs.lpi = Ls.lpi; qs.stages = Ls.stages;
            qs.nchunks = (pb.C + ts.bc - 1) / ts.bc;
            // split-C: the main tile's channel range per split, in the remainder tile's chunks
            qs.cper = zsplits > 1 ? q.cper * (t.bc / ts.bc) : qs.nchunks;
            qs.tx_in = (uint32_t)((size_t)box_imgs * ts.bc * Ls.rows_box * qs.pitch * sizeof(float));
            qs.solo = t.kg * t.tk / 4;                 // remainder CTAs per (slot tile, k tile): 4 channels each
            qs.tile0 = (int)grid.x / q.ktiles - rem;
            qs.trigger = 1;
            CUtensorMap tmap_s;
            memset(&tmap_s, 0, sizeof(tmap_s));
            if (!encode(&tmap_s, Ls, ts.bc)) return cudaErrorInvalidValue;
            e = dispatch_simt2(ts, pb.R, pb.S, true, in, kerp, kout, qs, tmap_s,
                               dim3((unsigned)(rem * q.ktiles * qs.solo), 1, (unsigned)zsplits), 128,
                               simt_smem_bytes(pb, ts), st);
            if (e != cudaSuccess) { err = std::string("SIMT remainder launch failed: ") + cudaGetErrorString(e); return e; }
            grid.x -= (unsigned)(rem * q.ktiles);
            q.nowait = 1; q.endwait = 1;
        }
        e = dispatch_simt2(t, pb.R, pb.S, L.tma, in, kerp, kout, q, tmap, grid, threads, smem, st);
    } else {
        e = dispatch_simt(t, in, kerp, kout, p, grid, threads, smem, st);
    }
    if (e != cudaSuccess) { err = std::string("SIMT kernel launch failed: ") + cudaGetErrorString(e); return e; }
    if (ev) cudaEventRecord(ev[2], st);
    if (zsplits > 1) {
        const int64_t tot = pb.out_elems();
        const int rblocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
        e = launch_pdl(reduce_splits, dim3(rblocks), 256, 0, st, (const float*)kout, out, tot, zsplits);
        if (e != cudaSuccess) { err = std::string("split-C reduce launch failed: ") + cudaGetErrorString(e); return e; }
        if (ev) cudaEventRecord(ev[3], st);
    }
    return cudaSuccess;
}

}  // namespace conv

// peaks.cu -- K5 bench-only kernels: the machine's own
// peaks, measured the way the paper measures the bandwidths its model uses
// ("per-core bandwidths ... obtained from synthetic benchmarks", PAPER.md:375,
// Sec. 7).  They feed the roofline denominators of bench.py and the selector's
// constants (csrc/peaks_measured.inc, written by scripts/measure_peaks.py).
// Not on the convolution path; libconv.so does not link this file.
//
//   probe_ffma      FP32 FFMA issue rate (register operands, 16 independent
//                   chains per thread) -> the "alu" peak of the SIMT path
//   probe_mma       tcgen05.mma issue rate from shared-memory operands
//                   (kind::f16 with bf16 inputs / kind::tf32, cta_group 1
//                   or 2, N = 256), no loads -> the tensor pipe's ceiling
//   probe_l2_bulk   L2 -> SMEM bandwidth of cp.async.bulk copies of an
//                   L2-resident buffer into a ring of smem stages (the
//                   DV_{L2->SMEM} level of the selector)
//   probe_l2_tiled  the same with 2-D tiled TMA boxes (128 rows x 128 B,
//                   128-B swizzle: the tensor kernel's operand loads)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/conv_probes.h"
#include "../csrc/sm100.cuh"

using namespace conv::sm100;

namespace {

// ---- FFMA -----------------------------------------------------------------
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float a0, float b0) {
    // register operands derived from the thread id: FFMA R, R, R, R (the SIMT
    // kernel's form), not the immediate / constant-bank forms
    const float a = a0 + 1e-7f * (float)(threadIdx.x & 7);
    const float b = b0 - 1e-7f * (float)(threadIdx.x & 3);
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = (float)(threadIdx.x + j) * 1e-3f;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += x[j];
    if (s == 1234.5678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;   // never true in practice; keeps the chains live
}

// FFMA2 (sm_100: two fp32 FMAs per lane in one instruction on a 64-bit
// register pair; fma.rn.f32x2): 8 pair chains, the multiplier pair and the
// broadcast scalar addend-free form the SIMT kernel uses (pair x scalar).
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, int iters, float a0, float b0) {
    const float a = a0 + 1e-7f * (float)(threadIdx.x & 7);
    const float b = b0 - 1e-7f * (float)(threadIdx.x & 3);
    unsigned long long ap, x[8];
    asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(a), "f"(b));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float lo = (float)(threadIdx.x + 2 * j) * 1e-3f, hi = (float)(threadIdx.x + 2 * j + 1) * 1e-3f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[j]) : "f"(lo), "f"(hi));
    }
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                unsigned long long bb;
                asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
                asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(x[j]) : "l"(ap), "l"(bb));
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += __int_as_float((int)x[j]) + __int_as_float((int)(x[j] >> 32));
    if (s == 1234.5678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- tcgen05.mma ------------------------------------------------------------
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <bool BF16, int CG>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int N = 256;
    constexpr uint32_t kA = 128 * 128, kB = (N / CG) * 128;     // one 128-B k-block of each operand
    // operands: random values in [-1, 1) (zeros would understate the power draw)
    for (uint32_t i = threadIdx.x; i < (kA + kB) / 4; i += blockDim.x) {
        const uint32_t h = hash32(i * 2654435761u + blockIdx.x);
        uint32_t v;
        if (BF16) {
            const uint32_t lo = 0x3f80u | (h & 0x7fu), hi = 0x3f80u | ((h >> 8) & 0x7fu);    // [1, 2)
            v = (lo ^ ((h >> 16) & 1u) << 15) | ((hi ^ ((h >> 17) & 1u) << 15) << 16);
        } else {
            v = (0x3f800000u | (h & 0x7fe000u)) ^ ((h >> 31) << 31);                         // tf32 in [1, 2)
        }
        reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        if (CG == 2) tmem_alloc_pair(&tslot, 512);
        else tmem_alloc(&tslot, 512);
    }
    fence_proxy_async_smem();                 // generic smem writes -> tensor core reads
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = make_idesc(BF16 ? 1u : 2u, 128 * CG, N);
    const uint64_t ad = make_sdesc(smem_u32(smem), 8 * 128, 2);
    const uint64_t bd = make_sdesc(smem_u32(smem + kA), 8 * 128, 2);
    if (warp == 0 && rank == 0) {
        const long long c0 = clock64();
        if (elect_one_sync()) {
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {           // 4 k steps of 32 B in the 128-B row
                    const uint32_t d = tmem + (uint32_t)((i & 1) * N);
                    if (CG == 2) {
                        if (BF16) mma_bf16_pair(d, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                        else mma_tf32_pair(d, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                    } else {
                        if (BF16) mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                        else mma_tf32(d, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                    }
                }
            }
            if (CG == 2) tc_commit_pair_mc(&bar, 0x3);
            else tc_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        const long long c1 = clock64();
        if (threadIdx.x == 0 && cycles) cycles[blockIdx.x] = (unsigned long long)(c1 - c0);
    } else if (CG == 2 && warp == 0) {
        mbar_wait(&bar, 0);                   // the leader's commit multicasts to both CTAs
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

// ---- L2 -> SMEM -----------------------------------------------------------
constexpr int kStages = 6;

// One thread per CTA keeps `kStages` copies of `chunk` bytes in flight; chunk
// i of CTA b reads offset ((b * 7919 + i * grid) * chunk) mod bytes.
__global__ void __launch_bounds__(32, 1) l2_bulk_kernel(const uint8_t* src, size_t bytes, uint32_t chunk, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    const size_t nchunks = bytes / chunk;
    auto issue = [&](int i, int s) {
        const size_t c = ((size_t)blockIdx.x * 7919u + (size_t)i * gridDim.x) % nchunks;
        mbar_arrive_expect_tx(&full[s], chunk);
        // <= 64 KB per bulk copy is plenty; split into 16-KB pieces
        for (uint32_t o = 0; o < chunk; o += 16384)
            bulk_load_g2s(smem + (size_t)s * chunk + o, src + c * chunk + o, min(16384u, chunk - o), &full[s]);
    };
    for (int s = 0; s < kStages && s < iters; ++s) issue(s, s);
    for (int i = 0; i < iters; ++i) {
        const int s = i % kStages;
        mbar_wait(&full[s], (uint32_t)(i / kStages) & 1);
        if (i + kStages < iters) issue(i + kStages, s);
    }
}

__global__ void __launch_bounds__(32, 1) l2_tiled_kernel(const __grid_constant__ CUtensorMap map, int rows, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages];
    if (threadIdx.x != 0) return;
    prefetch_tmap(&map);
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    constexpr uint32_t kBox = 128 * 128;      // 128 rows x 128 B
    constexpr int kPer = 2;                   // boxes per stage (32 KB)
    const int nbox = rows / 128;
    const uint64_t pol = policy_evict_normal();
    auto issue = [&](int i, int s) {
        mbar_arrive_expect_tx(&full[s], kPer * kBox);
        for (int j = 0; j < kPer; ++j) {
            const int b = (int)(((size_t)blockIdx.x * 7919u + (size_t)(i * kPer + j) * gridDim.x) % nbox);
            tma_load_2d(smem + ((size_t)s * kPer + j) * kBox, &map, &full[s], 0, b * 128, pol);
        }
    };
    for (int s = 0; s < kStages && s < iters; ++s) issue(s, s);
    for (int i = 0; i < iters; ++i) {
        const int s = i % kStages;
        mbar_wait(&full[s], (uint32_t)(i / kStages) & 1);
        if (i + kStages < iters) issue(i + kStages, s);
    }
}

template <typename F>
int set_smem(F kfn, size_t bytes) {
    return cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess ? 0 : -1;
}

}  // namespace

#define API extern "C" CONV_PROBE_API

API int probe_ffma(float* out, int blocks, int threads, int iters, void* stream) {
    if (!out || blocks < 1 || threads < 32 || threads > 256 || threads % 32 || iters < 1) return -1;
    ffma_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 0.999f, 1e-3f);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

API int probe_ffma2(float* out, int blocks, int threads, int iters, void* stream) {
    if (!out || blocks < 1 || threads < 32 || threads > 256 || threads % 32 || iters < 1) return -1;
    ffma2_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 0.999f, 1e-3f);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

API double probe_ffma_flops(int blocks, int threads, int iters) {
    return 2.0 * 16 * 8 * (double)iters * (double)blocks * threads;
}

API int probe_mma(int bf16, int cg, int grid, int iters, unsigned long long* cycles, void* stream) {
    if ((cg != 1 && cg != 2) || grid < cg || grid % cg || iters < 1) return -1;
    const size_t smem = 1024 + 128 * 128 + (256 / cg) * 128;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (bf16) {
        if (cg == 2) { set_smem(mma_kernel<true, 2>, smem); e = cudaLaunchKernelEx(&cfg, mma_kernel<true, 2>, iters, cycles); }
        else { set_smem(mma_kernel<true, 1>, smem); e = cudaLaunchKernelEx(&cfg, mma_kernel<true, 1>, iters, cycles); }
    } else {
        if (cg == 2) { set_smem(mma_kernel<false, 2>, smem); e = cudaLaunchKernelEx(&cfg, mma_kernel<false, 2>, iters, cycles); }
        else { set_smem(mma_kernel<false, 1>, smem); e = cudaLaunchKernelEx(&cfg, mma_kernel<false, 1>, iters, cycles); }
    }
    return e == cudaSuccess ? 0 : -2;
}

API double probe_mma_flops(int bf16, int cg, int grid, int iters) {
    // per CTA group and iteration: 4 MMAs of M = 128*cg, N = 256, K = 16 (bf16) / 8 (tf32)
    const double k = bf16 ? 16.0 : 8.0;
    return 2.0 * (grid / cg) * (double)iters * 4.0 * (128.0 * cg) * 256.0 * k;
}

API int probe_l2_bulk(const void* src, size_t bytes, int grid, unsigned chunk, int iters, void* stream) {
    if (!src || chunk == 0 || chunk % 16 || bytes < chunk || grid < 1 || iters < 1) return -1;
    const size_t smem = 1024 + (size_t)kStages * chunk;
    if (set_smem(l2_bulk_kernel, smem)) return -2;
    l2_bulk_kernel<<<grid, 32, smem, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint8_t*>(src), bytes,
                                                                          chunk, iters);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

typedef CUresult (*PFN_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

API int probe_l2_tiled(const void* src, size_t bytes, int grid, int iters, void* stream) {
    if (!src || bytes < 128 * 128 || grid < 1 || iters < 1) return -1;
    static PFN_tiled enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return -3;
        enc = reinterpret_cast<PFN_tiled>(fn);
    }
    const int rows = (int)(bytes / 128) / 128 * 128;
    CUtensorMap m;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(src), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -3;
    const size_t smem = 1024 + (size_t)kStages * 2 * 128 * 128;
    if (set_smem(l2_tiled_kernel, smem)) return -2;
    l2_tiled_kernel<<<grid, 32, smem, static_cast<cudaStream_t>(stream)>>>(m, rows, iters);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

API double probe_l2_tiled_bytes(int grid, int iters) { return (double)grid * iters * 2 * 128 * 128; }

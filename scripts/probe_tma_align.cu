// probe_tma_align.cu -- does a SWIZZLE_NONE 4-D TMA tile load accept a
// shared-memory destination that is only 16-B aligned (not 128-B)?  Loads a
// {16, 4, 1, 1} float box to smem offset `off` bytes for off in {0, 16, 32,
// 64, 80, 112, 128} and checks the values.  Study probe (r02b): decides
// whether the SIMT TMA layout may place image boxes at arbitrary 16-B
// offsets (bank-conflict-free image strides).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/probe_tma_align scripts/probe_tma_align.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int off) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    float* dst = reinterpret_cast<float*>(sm + off);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(b), "r"(256));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(b), "r"(0), "r"(0), "r"(0), "r"(0)
            : "memory");
    }
    __syncthreads();
    uint32_t ok = 0;
    long long t0 = clock64();
    while (!ok) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(b));
        if (clock64() - t0 > 2000000000ll) { out[0] = -1.f; return; }
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = dst[i];
}

int main() {
    float h[64], *d, *o;
    for (int i = 0; i < 64; ++i) h[i] = (float)(i + 1);
    cudaMalloc(&d, 256);
    cudaMalloc(&o, 256);
    cudaMemcpy(d, h, 256, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[4] = {16, 4, 1, 1};
    cuuint64_t str[3] = {64, 256, 256};
    cuuint32_t box[4] = {16, 4, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int offs[] = {0, 16, 32, 64, 80, 112, 128};
    for (int off : offs) {
        cudaMemset(o, 0, 256);
        k<<<1, 32, 2048>>>(m, o, off);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("off %3d: CUDA error %s\n", off, cudaGetErrorString(e)); return 2; }
        float g[64];
        cudaMemcpy(g, o, 256, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 64; ++i) bad += g[i] != h[i];
        printf("off %3d: %s (%d mismatches, out[0]=%g)\n", off, bad ? "WRONG" : "ok", bad, g[0]);
    }
    return 0;
}

// probe_shift.cu -- can a tcgen05 K-major swizzled A operand start at an
// arbitrary ROW of a shared-memory tile?  (SMEM halo reuse, SURVEY NEXT-1:
// the im2col operand of filter tap (r, s) is the input tile shifted by
// r*Win + s pixel rows; with shifted descriptors the tile would be loaded
// once instead of once per tap.)
//
// For each swizzle (64 B: 32 bf16 channels per row; 128 B: 64 channels),
// row shift t in [0, 8) and descriptor base-offset field bo in [0, 8): one
// M=128, N=32 bf16 MMA over the whole row (K = 32 or 64) with the A
// descriptor starting t rows into the tile; D is compared on the host with
// sum_k A[m + t][k] * B[n][k] (small integers: exact).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2101_09808_b200/csrc \
//        scripts/probe_shift.cu -o probe_shift && ./probe_shift
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"

using namespace conv::sm100;

constexpr int kRowsA = 160, kN = 32;

__host__ __device__ inline float aval(int m, int k) { return (float)(((m * 3 + k * 7) % 17) - 8); }
__host__ __device__ inline float bval(int n, int k) { return (float)(((n * 5 + k * 11) % 13) - 6); }

// byte offset of element (row, col) of a K-major tile with `rowb`-byte rows
// under the SWIZZLE_{64,128}B pattern (16-B chunk index XOR row bits)
__host__ __device__ inline uint32_t swz(int row, int col, int rowb) {
    const int chunk = (col * 2) / 16, within = (col * 2) % 16;
    const int x = rowb == 128 ? (row & 7) : ((row >> 1) & 3);
    return row * rowb + (((chunk ^ x) & (rowb / 16 - 1)) << 4) + within;
}

template <int ROWB>
__global__ void __launch_bounds__(128) probe(float* out) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    constexpr int K = ROWB / 2;                      // bf16 per row
    uint8_t* A = sm;
    uint8_t* B = sm + kRowsA * ROWB;                 // 1024-aligned (160 * 64 = 10240)
    for (int i = threadIdx.x; i < kRowsA * K; i += 128) {
        const int m = i / K, k = i % K;
        *reinterpret_cast<__nv_bfloat16*>(A + swz(m, k, ROWB)) = __float2bfloat16(aval(m, k));
    }
    for (int i = threadIdx.x; i < kN * K; i += 128) {
        const int n = i / K, k = i % K;
        *reinterpret_cast<__nv_bfloat16*>(B + swz(n, k, ROWB)) = __float2bfloat16(bval(n, k));
    }
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, 32);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t layout = ROWB == 128 ? 2u : 4u;
    constexpr uint32_t idesc = make_idesc(1u, 128, kN);
    uint32_t phase = 0;
    for (int t = 0; t < 8; ++t) {
        for (int bo = 0; bo < 8; ++bo) {
            if (threadIdx.x == 0) {
                const uint64_t ad = make_sdesc(smem_u32(A) + t * ROWB, 8 * ROWB, layout) | ((uint64_t)bo << 49);
                const uint64_t bd = make_sdesc(smem_u32(B), 8 * ROWB, layout);
                for (int kk = 0; kk < ROWB / 32; ++kk) mma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
                tc_commit(&bar);
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
            uint32_t v[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16), v);
            tmem_ld_wait();
            float* o = out + ((size_t)(t * 8 + bo) * 128 + warp * 32 + (threadIdx.x & 31)) * kN;
            for (int n = 0; n < kN; ++n) o[n] = __uint_as_float(v[n]);
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        }
    }
    if (warp == 0) tmem_dealloc(tmem, 32);
}

// timing: 256 back-to-back MMAs (M=128, N=64 / 256) from a descriptor
// starting `t` rows into the tile; clock64 span, one CTA
template <int ROWB, int NN>
__global__ void __launch_bounds__(128) probe_time(long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < (kRowsA + NN) * ROWB / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, NN < 32 ? 32 : NN);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    constexpr uint32_t layout = ROWB == 128 ? 2u : 4u;
    constexpr uint32_t idesc = make_idesc(1u, 128, NN);
    uint32_t phase = 0;
    for (int t = 0; t < 10; ++t) {
        if (threadIdx.x == 0) {
            const uint64_t bd = make_sdesc(smem_u32(sm + kRowsA * ROWB), 8 * ROWB, layout);
            const long long c0 = clock64();
            for (int i = 0; i < 256; ++i) {
                const int sh = (t < 8 ? t : (t == 8 ? 8 : 16)) + (i & 1) * 8;     // shifts t, t+8 alternate
                const uint64_t ad = make_sdesc(smem_u32(sm) + sh * ROWB, 8 * ROWB, layout);
                mma_bf16(tslot, ad, bd, idesc, 1);
            }
            tc_commit(&bar);
            mbar_wait(&bar, phase);
            cyc[t] = clock64() - c0;
        }
        phase ^= 1;
        __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, NN < 32 ? 32 : NN); }
}

template <int ROWB, int NN>
void run_time() {
    long long* d;
    cudaMalloc(&d, 16 * sizeof(long long));
    const size_t smem = 1024 + (kRowsA + NN) * ROWB;
    cudaFuncSetAttribute(probe_time<ROWB, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) probe_time<ROWB, NN><<<1, 128, smem>>>(d);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("swizzle %3dB N=%3d: cycles per MMA by start-row shift:", ROWB, NN);
    for (int t = 0; t < 10; ++t) printf(" %d:%.1f", t < 8 ? t : (t == 8 ? 8 : 16), h[t] / 256.0);
    printf("\n");
    cudaFree(d);
}

template <int ROWB>
void run() {
    constexpr int K = ROWB / 2;
    float* d;
    const size_t n = (size_t)64 * 128 * kN;
    cudaMalloc(&d, n * sizeof(float));
    const size_t smem = 1024 + kRowsA * ROWB + kN * ROWB;
    cudaFuncSetAttribute(probe<ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<ROWB><<<1, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("swizzle %d: %s\n", ROWB, cudaGetErrorString(e)); exit(1); }
    std::vector<float> h(n);
    cudaMemcpy(h.data(), d, n * sizeof(float), cudaMemcpyDeviceToHost);
    for (int t = 0; t < 8; ++t) {
        printf("swizzle %3dB shift %d rows: base_offset fields giving exact D:", ROWB, t);
        for (int bo = 0; bo < 8; ++bo) {
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int nn = 0; nn < kN; ++nn) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) ref += (double)aval(m + t, k) * bval(nn, k);
                    if (h[((size_t)(t * 8 + bo) * 128 + m) * kN + nn] != (float)ref) ++bad;
                }
            if (!bad) printf(" %d", bo);
        }
        printf("\n");
    }
    cudaFree(d);
}

int main() {
    run<64>();
    run<128>();
    run_time<64, 64>();
    run_time<64, 256>();
    run_time<128, 64>();
    run_time<128, 256>();
    return 0;
}

// probe_mma.cu -- microbenchmark: tcgen05.mma issue rate, SM clock under
// tensor load, and commit->mbarrier round trip.  One CTA per SM, operands in
// shared memory (contents irrelevant), no TMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2101_09808_b200/csrc probe_mma.cu -o probe_mma
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace conv::sm100;

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
    return pred != 0;
}

// MODE 0: back-to-back MMAs; 1: commit+wait every 4; 2: commit every 4 (no
// wait); 3: commit every 4 + try_wait on an already-complete barrier;
// 4: full producer/consumer ring (warp 1 = producer arriving immediately,
// thread 0 = MMA issuer) with STAGES stages; 5: as 4 but the whole MMA warp
// runs the loop and one elected lane issues.
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) probe(long long* cyc, unsigned long long* ns, int iters, const uint32_t* rnd) {
    extern __shared__ __align__(1024) uint8_t smem[];
    if (rnd) for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = rnd[i];
    __syncthreads();
    constexpr int STAGES = 6;
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, done_bar, full[STAGES], empty[STAGES];
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1); mbar_init(&done_bar, 1);
        for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) mbar_arrive(&done_bar);   // completes phase 0
    __syncthreads();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = make_idesc(1u, 128, N);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    if (MODE >= 4) {
        if (warp == 1 && lane == 0) {
            int st = 0; uint32_t ph = 0;
            for (int i = 0; i < iters; ++i) {
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive(&full[st]);
                if (++st == STAGES) { st = 0; ph ^= 1; }
            }
        }
        if (warp == 0 && (MODE == 5 || lane == 0)) {
            long long c0 = clock64();
            unsigned long long t0 = globaltimer_ns();
            int st = 0; uint32_t ph = 0;
            for (int i = 0; i < iters; ++i) {
                mbar_wait(&full[st], ph);
                tc_fence_after();
                if (MODE == 4 || elect_one()) {
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16(tmem, make_sdesc(a + kk * 32, 1024, 2), make_sdesc(b + kk * 32, 1024, 2), idesc, 1);
                    tc_commit(&empty[st]);
                }
                __syncwarp(MODE == 5 ? 0xffffffffu : 1u);
                if (++st == STAGES) { st = 0; ph ^= 1; }
            }
            if (MODE == 4 || elect_one()) tc_commit(&bar);
            mbar_wait(&bar, 0);
            if (lane == 0) {
                cyc[blockIdx.x] = clock64() - c0;
                ns[blockIdx.x] = globaltimer_ns() - t0;
            }
        }
    } else if (threadIdx.x == 0) {
        uint32_t phase = 0;
        long long c0 = clock64();
        unsigned long long t0 = globaltimer_ns();
        for (int i = 0; i < iters; ++i) {
            if (MODE == 3) { mbar_wait(&done_bar, 0); tc_fence_after(); }
            for (int kk = 0; kk < 4; ++kk) {
                mma_bf16(tmem, make_sdesc(a + kk * 32, 1024, 2), make_sdesc(b + kk * 32, 1024, 2), idesc, 1);
            }
            if (MODE == 1) {
                tc_commit(&bar);
                mbar_wait(&bar, phase);
                phase ^= 1;
            } else if (MODE >= 2) {
                tc_commit(&empty[i % STAGES]);
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, MODE == 1 ? phase : 0);
        long long c1 = clock64();
        unsigned long long t1 = globaltimer_ns();
        cyc[blockIdx.x] = c1 - c0;
        ns[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

__global__ void fill_random(uint32_t* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { uint32_t x = i * 2654435761u; x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
        // random bf16 pairs in [-1, 1): sign | exponent 0x3f.. | random mantissa
        p[i] = ((x & 0x80008000u) | 0x3f003f00u | ((x >> 1) & 0x007f007fu)); }
}

template <int N, int MODE>
void run(int sms, int iters) {
    long long* cyc; unsigned long long* ns;
    cudaMalloc(&cyc, sms * 8); cudaMalloc(&ns, sms * 8);
    size_t smem = 64 * 1024;
    cudaFuncSetAttribute(probe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    static uint32_t* rnd = nullptr;
    if (!rnd) { cudaMalloc(&rnd, 65536); fill_random<<<64, 256>>>(rnd, 16384); }
    const uint32_t* src = getenv("PROBE_RANDOM") ? rnd : nullptr;
    probe<N, MODE><<<sms, 128, smem>>>(cyc, ns, iters, src);   // warm
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<N, MODE><<<sms, 128, smem>>>(cyc, ns, iters, src);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h_c[256]; unsigned long long h_n[256];
    cudaMemcpy(h_c, cyc, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_n, ns, sms * 8, cudaMemcpyDeviceToHost);
    double cmax = 0, nmax = 0;
    for (int i = 0; i < sms; ++i) { if (h_c[i] > cmax) cmax = h_c[i]; if (h_n[i] > nmax) nmax = h_n[i]; }
    const double mmas = 4.0 * iters;
    const double flops = 2.0 * 128 * N * 16 * mmas * sms;
    printf("N=%d mode=%d err=%s: cycles/MMA=%.1f  clock=%.0f MHz  event=%.1f us  TFLOP/s(event)=%.0f\n",
           N, MODE, cudaGetErrorString(err), cmax / mmas, cmax / nmax * 1e3, ms * 1e3, flops / (ms * 1e-3) / 1e12);
    cudaFree(cyc); cudaFree(ns);
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<256, 0>(sms, 20000);
    run<256, 5>(sms, 20000);
    run<256, 0>(sms, 200000);
    return 0;
}

// repack.cu -- layout transforms of the tensor-core paths (SURVEY.md Sec. 8(a)
// rows a-2 / a-3).  The paper counts its own packing (Sec. 6)
// and "any time expended in internal layout transformations"
// in every measurement; conv_run launches these inside the timed region.
//
//   K1 ker: KCRS fp32 -> [K][R][S][Cp]   (c innermost = the GEMM K order of
//           the im2col A operand), channels C..Cp-1 zero.
//   K2 in : NCHW fp32 -> [N][Hin][Win][Cp] (NHWC; TMA im2col needs channels
//           innermost and 16-B aligned pixel strides), channels C..Cp-1 zero.
//
// Element conversion: TF32 path rounds to nearest, ties away (cvt.rna.tf32),
// BF16 path rounds to nearest even (cvt.rn.bf16x2).  Both are memory-bound
// (roofline: bytes / HBM bandwidth).
#include <cuda_bf16.h>
#include <stdint.h>

#include "internal.h"

namespace conv {

__device__ __forceinline__ float to_tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
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

// K1: one thread per output element (K*R*S*Cp <= 2^31).
template <bool BF16>
__global__ void __launch_bounds__(256) repack_ker_krsc(const float* __restrict__ ker,
                                                       typename Elem<BF16>::T* __restrict__ out,
                                                       int K, int C, int RS, int Cp) {
    const int64_t total = (int64_t)K * RS * Cp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % Cp);
        const int64_t krs = i / Cp;
        const int rs = (int)(krs % RS);
        const int64_t k = krs / RS;
        const float v = c < C ? __ldg(ker + (k * C + c) * RS + rs) : 0.0f;
        out[i] = Elem<BF16>::cvt(v);
    }
}

// K2: tiled transpose per image, 32 channels x 32 pixels per tile through
// shared memory (coalesced 128-B loads along pixels, coalesced stores along
// channels).  grid = (ceil(P/32), ceil(Cp/32), N), block = (32, 8).
template <bool BF16>
__global__ void __launch_bounds__(256) repack_in_nhwc(const float* __restrict__ in,
                                                      typename Elem<BF16>::T* __restrict__ out,
                                                      int C, int64_t P, int Cp) {
    __shared__ float tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t p0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    const int64_t n = blockIdx.z;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int c = c0 + ty + j;
        const int64_t p = p0 + tx;
        float v = 0.0f;
        if (c < C && p < P) v = __ldg(in + ((int64_t)n * C + c) * P + p);
        tile[ty + j][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t p = p0 + ty + j;
        const int c = c0 + tx;
        if (p < P && c < Cp) out[((int64_t)n * P + p) * Cp + c] = Elem<BF16>::cvt(tile[tx][ty + j]);
    }
}

cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev) {
    const int RS = pb.R * pb.S;
    const int64_t ktotal = (int64_t)pb.K * RS * Cp;
    const int kblocks = (int)((ktotal + 255) / 256 < 4096 ? (ktotal + 255) / 256 : 4096);
    const int64_t P = pb.Hin() * pb.Win();
    dim3 tgrid((unsigned)((P + 31) / 32), (unsigned)((Cp + 31) / 32), (unsigned)pb.N);
    dim3 tblock(32, 8);
    if (ev) cudaEventRecord(ev[0], st);
    if (bf16)
        repack_ker_krsc<true><<<kblocks, 256, 0, st>>>(ker, (__nv_bfloat16*)ker_ws, pb.K, pb.C, RS, Cp);
    else
        repack_ker_krsc<false><<<kblocks, 256, 0, st>>>(ker, (float*)ker_ws, pb.K, pb.C, RS, Cp);
    if (ev) cudaEventRecord(ev[1], st);
    if (bf16)
        repack_in_nhwc<true><<<tgrid, tblock, 0, st>>>(in, (__nv_bfloat16*)in_ws, pb.C, P, Cp);
    else
        repack_in_nhwc<false><<<tgrid, tblock, 0, st>>>(in, (float*)in_ws, pb.C, P, Cp);
    if (ev) cudaEventRecord(ev[2], st);
    return cudaGetLastError();
}

}  // namespace conv

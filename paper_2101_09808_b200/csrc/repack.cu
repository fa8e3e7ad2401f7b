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

// K1 (generic): one thread per output element (K*R*S*Cp <= 2^31).
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

// K1 (fast): one CTA per output channel k.  The k-th filter (C*R*S
// contiguous floats) is staged in shared memory with coalesced loads, then
// written c-innermost with coalesced stores.  Used when C*R*S*4 <= 48 KB.
template <bool BF16>
__global__ void __launch_bounds__(256) repack_ker_krsc_smem(const float* __restrict__ ker,
                                                            typename Elem<BF16>::T* __restrict__ out,
                                                            int C, int RS, int Cp) {
    extern __shared__ float filt[];
    const int64_t k = blockIdx.x;
    const int crs = C * RS;
    const float* src = ker + k * crs;
    for (int i = threadIdx.x; i < crs; i += blockDim.x) filt[i] = __ldg(src + i);
    __syncthreads();
    typename Elem<BF16>::T* dst = out + k * (int64_t)RS * Cp;
    for (int i = threadIdx.x; i < RS * Cp; i += blockDim.x) {
        const int rs = i / Cp;
        const int c = i - rs * Cp;
        dst[i] = Elem<BF16>::cvt(c < C ? filt[c * RS + rs] : 0.0f);
    }
}

// K2: tiled transpose per image, 64 channels x 64 pixels per CTA through a
// padded shared-memory tile.  Loads are float4 along pixels (when the pixel
// count P is a multiple of 4; scalar otherwise), stores are 16-B vectors of
// 8 bf16 / 4 fp32 consecutive channels of one pixel, so both sides move
// full 128-B lines.  grid = (ceil(P/64), ceil(Cp/64), N), block = 256.
template <bool BF16>
__global__ void __launch_bounds__(256) repack_in_nhwc(const float* __restrict__ in,
                                                      typename Elem<BF16>::T* __restrict__ out,
                                                      int C, int64_t P, int Cp) {
    __shared__ float tile[64][65];
    const int tid = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * 64;
    const int c0 = blockIdx.y * 64;
    const int64_t n = blockIdx.z;
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
    typename Elem<BF16>::T* dst = out + n * P * Cp;
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
                    const __nv_bfloat162 b = __floats2bfloat162_rn(tile[cq + 2 * j][pl], tile[cq + 2 * j + 1][pl]);
                    w[j] = *reinterpret_cast<const uint32_t*>(&b);
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
}

cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev) {
    const int RS = pb.R * pb.S;
    const int64_t P = pb.Hin() * pb.Win();
    if (ev) cudaEventRecord(ev[0], st);
    const size_t filt_bytes = (size_t)pb.C * RS * sizeof(float);
    if (filt_bytes <= 48 * 1024) {
        if (bf16)
            repack_ker_krsc_smem<true><<<pb.K, 256, filt_bytes, st>>>(ker, (__nv_bfloat16*)ker_ws, pb.C, RS, Cp);
        else
            repack_ker_krsc_smem<false><<<pb.K, 256, filt_bytes, st>>>(ker, (float*)ker_ws, pb.C, RS, Cp);
    } else {
        const int64_t ktotal = (int64_t)pb.K * RS * Cp;
        const int kblocks = (int)((ktotal + 255) / 256 < 4096 ? (ktotal + 255) / 256 : 4096);
        if (bf16)
            repack_ker_krsc<true><<<kblocks, 256, 0, st>>>(ker, (__nv_bfloat16*)ker_ws, pb.K, pb.C, RS, Cp);
        else
            repack_ker_krsc<false><<<kblocks, 256, 0, st>>>(ker, (float*)ker_ws, pb.K, pb.C, RS, Cp);
    }
    if (ev) cudaEventRecord(ev[1], st);
    dim3 tgrid((unsigned)((P + 63) / 64), (unsigned)((Cp + 63) / 64), (unsigned)pb.N);
    if (bf16)
        repack_in_nhwc<true><<<tgrid, 256, 0, st>>>(in, (__nv_bfloat16*)in_ws, pb.C, P, Cp);
    else
        repack_in_nhwc<false><<<tgrid, 256, 0, st>>>(in, (float*)in_ws, pb.C, P, Cp);
    if (ev) cudaEventRecord(ev[2], st);
    return cudaGetLastError();
}

}  // namespace conv

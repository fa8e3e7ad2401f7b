// repack.cu -- layout transforms of the tensor-core paths (SURVEY.md Sec. 8(a)
// rows a-2 / a-3).  The paper counts its own packing (Sec. 6)
// and "any time expended in internal layout transformations"
// in every measurement; conv_run launches these inside the timed region.
//
//   K1 ker: KCRS fp32 -> [K][R][S][Cp]   (c innermost = the GEMM K order of
//           the im2col A operand), channels C..Cp-1 zero.
//   K2 in : NCHW fp32 -> [N][Hin][Win][Cp] (NHWC; TMA im2col needs channels
//           innermost and 16-B aligned pixel strides), channels C..Cp-1 zero.
// Both run in ONE launch (repack_all).
//
// Element conversion: TF32 path rounds to nearest, ties away (cvt.rna.tf32),
// BF16 path rounds to nearest even (cvt.rn.bf16x2).  Both are memory-bound
// (roofline: bytes / HBM bandwidth).
#include <cuda_bf16.h>
#include <stdint.h>

#include <algorithm>

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

// One launch performs both layout transforms (PAPER.md:371 packing; the
// two are independent, so merging them removes a kernel boundary):
//   CTAs [0, n_ker)          K1: Ker KCRS fp32 -> [K][R][S][Cp], one CTA per
//                            (k, chunk of `cc` channels): the chunk's cc*R*S
//                            contiguous floats are staged in shared memory with
//                            coalesced loads, then written c-innermost with
//                            coalesced stores; channels C..Cp-1 are zero.
//   CTAs [n_ker, n_ker+n_in) K2: NCHW fp32 -> NHWC, one CTA per (image,
//                            64-channel block, 64-pixel block) through a padded
//                            64x65 tile: float4 loads along pixels (scalar when
//                            the pixel count is not a multiple of 4), 16-B
//                            stores of 8 bf16 / 4 fp32 consecutive channels.
struct RepackGeom {
    int C, Cp, RS, cc, ker_chunks;   // K1
    int64_t P;                       // K2: pixels per image
    int ptiles, ctiles;              // K2 tile grid per image
    int n_ker;                       // number of K1 CTAs
};

template <bool BF16>
__global__ void __launch_bounds__(256) repack_all(const float* __restrict__ in, const float* __restrict__ ker,
                                                  typename Elem<BF16>::T* __restrict__ in_ws,
                                                  typename Elem<BF16>::T* __restrict__ ker_ws, const RepackGeom g) {
    extern __shared__ float sm[];
    const int tid = threadIdx.x;
    // let the dependent main kernel (launched with programmatic stream
    // serialization) start its prologue as SMs free up; it waits for this
    // grid's completion (griddepcontrol.wait) before reading the workspace
    asm volatile("griddepcontrol.launch_dependents;");
    if ((int)blockIdx.x < g.n_ker) {
        // ---- K1 ----
        const int64_t k = blockIdx.x / g.ker_chunks;
        const int c0 = (blockIdx.x % g.ker_chunks) * g.cc;
        const int c1 = min(c0 + g.cc, g.Cp);
        const int cload = max(0, min(c1, g.C) - c0);
        const float* src = ker + (k * g.C + c0) * g.RS;
        for (int i = tid; i < cload * g.RS; i += 256) sm[i] = __ldg(src + i);
        __syncthreads();
        typename Elem<BF16>::T* dst = ker_ws + k * (int64_t)g.RS * g.Cp;
        const int width = c1 - c0;
        for (int i = tid; i < g.RS * width; i += 256) {
            const int rs = i / width;
            const int c = c0 + (i - rs * width);
            dst[(int64_t)rs * g.Cp + c] = Elem<BF16>::cvt(c < g.C ? sm[(c - c0) * g.RS + rs] : 0.0f);
        }
        return;
    }
    // ---- K2 ----
    float (*tile)[65] = reinterpret_cast<float (*)[65]>(sm);
    int b = blockIdx.x - g.n_ker;
    const int pt = b % g.ptiles;
    b /= g.ptiles;
    const int ct = b % g.ctiles;
    const int64_t n = b / g.ctiles;
    const int64_t P = g.P;
    const int C = g.C, Cp = g.Cp;
    const int64_t p0 = (int64_t)pt * 64;
    const int c0 = ct * 64;
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
    typename Elem<BF16>::T* dst = in_ws + n * P * Cp;
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
                    const __nv_bfloat162 bb = __floats2bfloat162_rn(tile[cq + 2 * j][pl], tile[cq + 2 * j + 1][pl]);
                    w[j] = *reinterpret_cast<const uint32_t*>(&bb);
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
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev, bool with_in) {
    RepackGeom g;
    g.C = pb.C;
    g.Cp = Cp;
    g.RS = pb.R * pb.S;
    // channels per K1 CTA so that the staged slice is <= 32 KB (at least 1)
    g.cc = std::max(1, std::min(Cp, (int)(32768 / (4 * g.RS))));
    g.ker_chunks = (Cp + g.cc - 1) / g.cc;
    g.n_ker = pb.K * g.ker_chunks;
    g.P = pb.Hin() * pb.Win();
    g.ptiles = (int)((g.P + 63) / 64);
    g.ctiles = (Cp + 63) / 64;
    const int64_t n_in = with_in ? (int64_t)g.ptiles * g.ctiles * pb.N : 0;   // fused: Ker only
    const int64_t grid = g.n_ker + n_in;
    if (grid >= (1ll << 31)) return cudaErrorInvalidValue;
    const size_t smem = std::max<size_t>(64 * 65 * sizeof(float), (size_t)g.cc * g.RS * sizeof(float));
    if (smem > 48 * 1024) {   // very large R*S: one channel per K1 CTA still needs > 48 KB
        cudaError_t e = bf16 ? cudaFuncSetAttribute(repack_all<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(repack_all<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (ev) cudaEventRecord(ev[0], st);
    if (bf16)
        repack_all<true><<<(unsigned)grid, 256, smem, st>>>(in, ker, (__nv_bfloat16*)in_ws, (__nv_bfloat16*)ker_ws, g);
    else
        repack_all<false><<<(unsigned)grid, 256, smem, st>>>(in, ker, (float*)in_ws, (float*)ker_ws, g);
    if (ev) cudaEventRecord(ev[1], st);
    return cudaGetLastError();
}

}  // namespace conv

/*
 * conv_probes.h -- C ABI of libconv_probes.so: the bench-only peak probes
 * (SURVEY.md Sec. 2c, K5).  The paper's model divides each memory level's data
 * volume by that level's bandwidth and takes the bandwidths from synthetic
 * benchmarks on the machine itself (Sec. 7; PAPER.md:296-300,
 * Sec. 5); these kernels are that step for B200.  scripts/measure_peaks.py
 * times them (CUDA events on the caller's stream) and writes
 * profiles/peaks_measured.json and csrc/peaks_measured.inc.
 *
 * Not part of the convolution path (include/conv.h).  Every launcher is
 * asynchronous on `stream` (cudaStream_t as void*, NULL = legacy default),
 * returns 0 on success, -1 for an invalid argument (nothing launched), -2 if
 * the launch failed and -3 if a driver entry point / tensor map failed.
 */
#ifndef CONV_PROBES_H_
#define CONV_PROBES_H_

#include <stddef.h>

#if defined(__GNUC__)
#define CONV_PROBE_API __attribute__((visibility("default")))
#else
#define CONV_PROBE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* FP32 FFMA issue rate: `blocks` x `threads` (32..256, multiple of 32)
 * threads, each running 16 independent register-operand FFMA chains for
 * 8 * iters steps.  `out` (device, blocks*threads floats) is written only in
 * a never-taken branch.  probe_ffma_flops = 2 * 16 * 8 * iters * blocks *
 * threads, the FLOPs one launch executes. */
CONV_PROBE_API int probe_ffma(float* out, int blocks, int threads, int iters, void* stream);
CONV_PROBE_API double probe_ffma_flops(int blocks, int threads, int iters);

/* FFMA2 (fma.rn.f32x2: two fp32 FMAs per lane and instruction, sm_100):
 * 8 register-pair chains x 8 * iters steps, pair x broadcast-scalar
 * operands (the SIMT kernel's form); same FLOPs per launch as probe_ffma
 * with the same arguments. */
CONV_PROBE_API int probe_ffma2(float* out, int blocks, int threads, int iters, void* stream);

/* tcgen05.mma issue rate from shared-memory operands (no loads): `grid` CTAs
 * (a multiple of cg; cluster of cg), each CTA group issuing 4 * iters MMAs of
 * M = 128*cg, N = 256, K = 16 (bf16 != 0, kind::f16 with bf16 inputs) or
 * K = 8 (kind::tf32), fp32 accumulation in TMEM.  cycles (device, optional,
 * grid entries): the issuing CTA's clock64 span.  probe_mma_flops = the
 * FLOPs of one launch. */
CONV_PROBE_API int probe_mma(int bf16, int cg, int grid, int iters, unsigned long long* cycles, void* stream);
CONV_PROBE_API double probe_mma_flops(int bf16, int cg, int grid, int iters);

/* L2 -> shared memory bandwidth: `grid` CTAs, one thread each, keep 6 copies
 * of `chunk` bytes (multiple of 16; 6*chunk must fit shared memory) in
 * flight with cp.async.bulk from the device buffer src[0, bytes) (keep it
 * L2-resident: bytes well below the 126 MB L2, read once beforehand); each CTA
 * moves iters * chunk bytes. */
CONV_PROBE_API int probe_l2_bulk(const void* src, size_t bytes, int grid, unsigned chunk, int iters, void* stream);

/* The same with 2-D tiled TMA loads (cp.async.bulk.tensor, 128 rows x 128 B
 * boxes, 128-B swizzle -- the tensor kernel's operand-load shape), two boxes
 * per stage; probe_l2_tiled_bytes = bytes one launch moves. */
CONV_PROBE_API int probe_l2_tiled(const void* src, size_t bytes, int grid, int iters, void* stream);
CONV_PROBE_API double probe_l2_tiled_bytes(int grid, int iters);

#ifdef __cplusplus
}
#endif

#endif /* CONV_PROBES_H_ */

/*
 * conv.h -- C ABI of the B200-native direct-convolution library (libconv.so).
 *
 * Operation (Sec. 1, Eq. 1 of Li et al., ASPLOS'21):
 *
 *     Out[n,k,h,w] = sum_{c<C, r<R, s<S} In[n,c,h+r,w+s] * Ker[k,c,r,s]
 *
 * no padding, fp32 tensors, In/Out NCHW and Ker KCRS
 * (Sec. 9: "All input and output tensors were stored in NCHW
 * layout and all kernel tensors were stored in KCRS layout").  H and W are the
 * OUTPUT extents (the loop extents N_h, N_w of Listing 2);
 * the input is (H+R-1) x (W+S-1) (Sec. 3.1).  conv_run
 * OVERWRITES Out (Eq. 1 is "=", reading R4).  Plans made with
 * conv_plan_create_strided use stride U (PAPER.md:201 footnote 1: the method
 * "is applicable to the general case" of strided convolution; Table 1,
 * PAPER.md:439, marks the stride-2 layers with *):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+r,U*w+s] * Ker[k,c,r,s]
 *
 * with explicit INPUT extents Hin x Win and H = (Hin-R)/U + 1 (floor).
 * conv_plan_create_dilated adds dilation D (the footnote's other case):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+D*r,U*w+D*s] * Ker[k,c,r,s]
 *
 * with H = (Hin - D*(R-1) - 1)/U + 1 (floor), likewise W.
 * conv_plan_create_padded adds zero padding ph (rows, top and bottom) and pw
 * (columns, left and right) -- the "same"-padded layers of real networks
 * (Eq. 1 itself has none, R3):
 *
 *     Out[n,k,h,w] = sum_{c,r,s} In[n,c,U*h+D*r-ph,U*w+D*s-pw] * Ker[k,c,r,s]
 *
 * with In = 0 outside [0,Hin) x [0,Win) and H = (Hin + 2ph - D*(R-1) - 1)/U + 1.
 * Internal layout
 * transforms are part of every conv_run, as the paper counts them
 * (PAPER.md:371).
 *
 * Conventions (all functions):
 *   - Plain C types only.  Device pointers are CUDA device pointers on the
 *     device that was current when the plan was created.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every conv_status-returning call returns CONV_OK (0) or an error code;
 *     conv_last_error() then returns a thread-local, NUL-terminated message
 *     (static storage, valid until the next failing call on that thread).
 *   - Error classes follow SPEC.md:552's exit-code classes: 1 = invalid
 *     argument / usage, 2 = infeasible request; 3, 4 add CUDA and device
 *     failures.  There is no CPU fallback: on a machine without an sm_100
 *     device, conv_plan_create fails with CONV_ERR_UNSUPPORTED_DEVICE.
 *   - Thread safety: a plan is immutable after create / set_path / set_tile.
 *     conv_run may be called concurrently on one plan from several host
 *     threads / streams if each call has its own workspace.  Plans whose main
 *     kernel needs all of its CTAs resident at once (describe: "fuse":1 or
 *     "splits">1) are serialised per device by the library: such a conv_run
 *     waits on the device for the previous one's main kernel (an internal
 *     event), so two of them never share the SMs.  Inside CUDA-graph capture
 *     that wait is not inserted; do not replay two graphs holding such plans
 *     concurrently on one device.
 */
#ifndef CONV_H_
#define CONV_H_

#include <stddef.h>

#if defined(__GNUC__)
#define CONV_API __attribute__((visibility("default")))
#else
#define CONV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct conv_plan conv_plan; /* opaque, owned by the library */

typedef enum {
    CONV_OK = 0,
    CONV_ERR_INVALID_ARGUMENT = 1,  /* extent < 1, size overflow, NULL/misaligned pointer */
    CONV_ERR_INFEASIBLE = 2,        /* no tile fits the hardware limits for the requested path */
    CONV_ERR_CUDA = 3,              /* a CUDA runtime/driver call or launch failed */
    CONV_ERR_UNSUPPORTED_DEVICE = 4 /* no device, or the current device is not sm_100 */
} conv_status;

typedef enum {
    CONV_PATH_AUTO = 0,      /* the faster (modeled) of the two FP32-precision paths: FP32_SIMT, FP32_TC */
    CONV_PATH_FP32_SIMT = 1, /* FP32 FFMA direct convolution on native NCHW In (Ker packed) */
    CONV_PATH_TF32 = 2,      /* tcgen05 implicit GEMM, inputs rounded to TF32 (RNA), fp32 accumulate */
    CONV_PATH_BF16 = 3,      /* tcgen05 implicit GEMM, inputs rounded to BF16 (RNE), fp32 accumulate */
    CONV_PATH_FP32_TC = 4    /* FP32-accurate on the tensor cores: every fp32 input split EXACTLY into three
                                bf16 pieces x = x0 + x1 + x2 (RNE remainders); the products x_i * y_j with
                                i + j <= 2 (6 pairs; dropped terms < 3 * 2^-24 |x*y|), or all 9 with the tile
                                key split=9 (every product exact), accumulated in fp32 by the tcgen05 bf16
                                kernel over npairs x the channels (reading R15) */
} conv_path;

/* ---- plans ------------------------------------------------------------- */

/* Create a plan for Eq. 1 with batch N, output channels K, input channels C,
 * OUTPUT extents H x W and kernel R x S (In is N x C x (H+R-1) x (W+S-1)).
 * Binds to the current CUDA device, queries its attributes and runs the tile
 * selector (Sec. 5 min-max,
 * PAPER.md:383-419 Alg. 1).  Returns NULL on error (conv_last_error()):
 * INVALID_ARGUMENT if an extent is < 1 ("all extents >= 1") or a
 * tensor has >= 2^31 elements; UNSUPPORTED_DEVICE without an sm_100 device. */
CONV_API conv_plan* conv_plan_create(int N, int K, int C, int H, int W, int R, int S);

/* Strided plan: input extents Hin x Win (as PAPER.md:439 Table 1 lists them),
 * kernel R x S, stride U >= 1 on both axes; output H = (Hin-R)/U + 1,
 * W = (Win-S)/U + 1 (input rows/columns past the last full window are not
 * read).  In is N x C x Hin x Win.  With U = 1 and Hin = H+R-1 it is the
 * same plan as conv_plan_create.  Paths: the tensor-core paths (TMA im2col
 * traversal stride U, U <= 8) and FP32 SIMT v1; SIMT v2 needs U = 1.
 * Errors as conv_plan_create, plus INVALID_ARGUMENT if U < 1 or the input is
 * smaller than the kernel. */
CONV_API conv_plan* conv_plan_create_strided(int N, int K, int C, int Hin, int Win, int R, int S, int U);

/* Strided and dilated plan (PAPER.md:201 footnote 1): as
 * conv_plan_create_strided plus dilation D >= 1 on both axes -- tap (r, s)
 * reads input row U*h + D*r, column U*w + D*s; H = (Hin - D*(R-1) - 1)/U + 1,
 * W = (Win - D*(S-1) - 1)/U + 1.  D = 1 is conv_plan_create_strided.
 * Paths: the tensor-core paths (tap (r, s) is the TMA im2col offset
 * (D*s, D*r); needs D*(R-1), D*(S-1) <= 128) and FP32 SIMT v1; SIMT v2
 * needs U = D = 1.  Errors as conv_plan_create_strided, plus
 * INVALID_ARGUMENT if D < 1 or the input is smaller than the dilated kernel
 * (D*(R-1)+1) x (D*(S-1)+1). */
CONV_API conv_plan* conv_plan_create_dilated(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D);

/* Padded, strided and dilated plan (the general form above): zero padding
 * ph >= 0 rows above and below, pw >= 0 columns left and right; H = (Hin +
 * 2ph - D*(R-1) - 1)/U + 1, W likewise.  ph = pw = 0 is
 * conv_plan_create_dilated.  The padding is never materialised: the tensor
 * paths' TMA im2col box starts at (-pw, -ph) and TMA zero-fills the
 * out-of-bounds taps (needs ph, pw <= 128 and pad - D*(R-1) in [-128, 127]);
 * FP32 SIMT v1 zero-fills its smem halo; SIMT v2 needs no padding.  Errors
 * as conv_plan_create_dilated, plus INVALID_ARGUMENT if ph or pw < 0 or the
 * padded input is smaller than the dilated kernel. */
CONV_API conv_plan* conv_plan_create_padded(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D,
                                            int ph, int pw);

/* A plan for a described (not present) device: `sms` SMs, `smem_optin` bytes
 * of opt-in shared memory per block, `l2_bytes` of L2.  Runs the same
 * selector; the plan can be described but not run (conv_run returns
 * CONV_ERR_UNSUPPORTED_DEVICE).  For the selector's CPU tests and offline
 * studies.  NULL on invalid arguments. */
CONV_API conv_plan* conv_plan_create_offline(int N, int K, int C, int H, int W, int R, int S,
                                             int sms, size_t smem_optin, size_t l2_bytes);
/* Offline variant of conv_plan_create_strided (same arguments as above). */
CONV_API conv_plan* conv_plan_create_strided_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                     int sms, size_t smem_optin, size_t l2_bytes);
/* Offline variant of conv_plan_create_dilated (same arguments as above). */
CONV_API conv_plan* conv_plan_create_dilated_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                     int D, int sms, size_t smem_optin, size_t l2_bytes);
/* Offline variant of conv_plan_create_padded (same arguments as above). */
CONV_API conv_plan* conv_plan_create_padded_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                    int D, int ph, int pw, int sms, size_t smem_optin,
                                                    size_t l2_bytes);

/* Force a path (default AUTO) and re-run the selector for it.
 * INFEASIBLE if no candidate of that path fits (e.g. R or S > 128 on the
 * tensor paths: TMA im2col offsets are limited to [-128, 127]). */
CONV_API conv_status conv_plan_set_path(conv_plan* plan, conv_path path);

/* Force a tiling (tests / the selector-validation study).  `spec` is a
 * comma-separated key=value list; keys for the tensor paths: bn (32, 64,
 * 128, 192, 256), cg (1 or 2: CTA pair), kbs (k-blocks per stage: 1-4, 6-9),
 * stages, splits (split-K count, 1-16), fuse (0/1: in-kernel In transform),
 * pre_c (fused prologue channels), expand (0/1: tiny-C tap expansion -- the
 * transform writes each output pixel's R*S*C taps as channels and the
 * kernel runs the equivalent 1x1 problem; automatic when C*elem <= 16 B and
 * R*S >= 4, and then free of the TMA limits stated above), split (FP32_TC:
 * 6 or 9 bf16 piece pairs, default 6), halo (0/1: the halo kernel -- the
 * input tile staged once per CTA in shared memory, the filter taps as
 * shifted tcgen05 descriptors; stride 1, dilation 1, no padding,
 * C*elem <= 128 B, K <= 256; only on request); for the SIMT
 * path: ver, tk, tw, kg, pw, tn, th, bc, splits (split-C), flat (0/1: v2
 * row mode over whole images, TW = W in {7, 14}, Win % 4 == 0: each CTA's
 * 32*pw lanes take consecutive (image, row) slots of the flattened batch,
 * so no lane is padding; tn is then the images one In box spans and th = H),
 * rem (0/1, flat tiles, default 1: the slot tiles that would start a mostly
 * empty extra CTA per SM run as a second, small grid of 4-warp CTAs beside
 * the main grid -- same arithmetic per output, bit-identical results; with
 * split-C it takes the same per-split channel ranges and partial slabs;
 * describe() reports the slot tiles it takes as tile.rem).
 * Unspecified keys keep the
 * selector's choice.  NULL or "" restores the selector's choice.
 * INVALID_ARGUMENT on a malformed spec, INFEASIBLE if the tile exceeds
 * SMEM/TMEM/register capacity (Eq. 4, per level). */
CONV_API conv_status conv_plan_set_tile(conv_plan* plan, const char* spec);

/* Bytes of device workspace conv_run needs: the NHWC In / KRSC Ker buffers of
 * the tensor paths (FP32_TC: of the bf16 pieces, 6 pair blocks of the
 * channels; halo plans: only the per-tap Ker image), the packed
 * [K/BKo][C][R][S][BKo] Ker of the SIMT path, plus the fused transform's
 * chunk flags / split-K partial slabs when the plan uses them.
 * Caller allocates, 256-B aligned. */
CONV_API size_t conv_plan_workspace_bytes(const conv_plan* plan);

/* Number of timed stages of one conv_run (conv_run_events records one event
 * around each): 2 (one layout transform launch + the main kernel), 3 for
 * FP32 SIMT plans with a split-C reduction (the splits' partial outputs
 * summed in split order by a third kernel).  An FP32 SIMT flat plan with a
 * remainder grid (tile.rem > 0 in describe()) launches that grid and the main
 * grid as one stage: two launches that run side by side. */
CONV_API int conv_plan_num_kernels(const conv_plan* plan);

/* Path the plan will run (never AUTO after create). */
CONV_API conv_path conv_plan_path(const conv_plan* plan);

/* Write a JSON description (path, tiles, modeled data volume per level and
 * bandwidth-scaled costs, roofline) into buf (NUL-terminated, truncated to
 * cap).  Returns the number of bytes needed excluding the NUL, or -1. */
CONV_API int conv_plan_describe(const conv_plan* plan, char* buf, size_t cap);

/* NULL-safe. */
CONV_API void conv_plan_destroy(conv_plan* plan);

/* ---- execution ---------------------------------------------------------- */

/* Out = Eq. 1 (In, Ker), asynchronously on `stream`.
 *   in:  N*C*(H+R-1)*(W+S-1) fp32, NCHW, contiguous, 16-B aligned
 *   ker: K*C*R*S fp32, KCRS, contiguous, 16-B aligned
 *   out: N*K*H*W fp32, NCHW, contiguous, 16-B aligned; overwritten; must not
 *        alias in, ker or workspace
 *   workspace: >= conv_plan_workspace_bytes(plan) bytes, 256-B aligned
 *        (may be NULL when that is 0).
 * Returns INVALID_ARGUMENT on NULL/misaligned pointers, CUDA on a launch
 * error.  Asynchronous faults surface at the caller's next synchronisation. */
CONV_API conv_status conv_run(const conv_plan* plan, const float* in, const float* ker,
                     float* out, void* workspace, void* stream);

/* As conv_run, and records caller-created cudaEvent_t handles (passed as
 * void*) on `stream` around each kernel: events[0] before the first kernel,
 * events[i] after kernel i (i = 1..num_kernels).  n_events must be
 * conv_plan_num_kernels(plan) + 1.  Used by bench.py to time the dominant
 * kernel on the stream it is launched on. */
CONV_API conv_status conv_run_events(const conv_plan* plan, const float* in, const float* ker,
                            float* out, void* workspace, void* stream,
                            void* const* events, int n_events);

/* Device bytes conv_run_host needs: In + Ker + Out device copies + workspace. */
CONV_API size_t conv_plan_host_run_bytes(const conv_plan* plan);

/* End-to-end call with HOST buffers (pinned for overlap; pageable works but
 * synchronises): copies in/ker host->device into `device_buffer`
 * (>= conv_plan_host_run_bytes, 256-B aligned), runs the plan's kernels,
 * copies Out device->host.  Large batches are pipelined over image chunks
 * (upload of chunk j+1, kernels of chunk j and download of chunk j-1 overlap
 * on three streams the plan owns; one cudaMemcpyAsync per tensor chunk); the
 * chunks are chosen once per plan by simulating the pipeline on the
 * selector's model (conv_plan_describe "host_pipeline").  Everything starts
 * after the work already queued on `stream`, and `stream` waits for all of
 * it: the call is asynchronous, out_host is valid after `stream`
 * synchronises.  Results are bit-identical to conv_run.  Concurrent calls on
 * one plan are serialised (the pipeline resources are per plan). */
CONV_API conv_status conv_run_host(const conv_plan* plan, const float* in_host, const float* ker_host,
                          float* out_host, void* device_buffer, void* stream);

/* Thread-local message for the last failing call on this thread ("" if none). */
CONV_API const char* conv_last_error(void);

/* Thread-local status code of that failing call (CONV_OK if none) -- how a
 * caller tells INVALID_ARGUMENT / INFEASIBLE / UNSUPPORTED_DEVICE apart when
 * a conv_plan_create* call returns NULL. */
CONV_API conv_status conv_last_status(void);

/* Library version string, e.g. "0.1.0 sm_100a". */
CONV_API const char* conv_version(void);

/* ---- the tile selector's data-movement model (host only, no device) ------ */

/* Sec. 3.2's data volume for single-level tiling of Eq. 1
 * with tile-loop permutation perm[0..6] (outermost first; iterator ids
 * n=0,k=1,c=2,r=3,s=4,h=5,w=6), problem extents Nx[7] and tile sizes T[7]
 * (same id order; 1 <= T <= N; trip counts ceil(N/T)).  Writes the In, Ker,
 * Out volumes (words) to dv[0..2] and returns their sum; Out carries the
 * paper's factor 2 (read + write).  Returns -1 on bad input. */
CONV_API double conv_model_dv(const int perm[7], const double Nx[7], const double T[7], double dv[3]);

/* Sec. 2.2's matmul model (Eq. 3): C[i][j] += A[i][k]*B[k][j]
 * tiled by T[3] with tile-loop permutation perm[0..2] (ids i=0,j=1,k=2).
 * Returns the total data volume (C counted twice), -1 on bad input. */
CONV_API double conv_model_dv_matmul(const int perm[3], const double Nx[3], const double T[3]);

/* Eq. 4 left-hand side: the tile footprint of In + Ker + Out. */
CONV_API double conv_model_footprint(const double T[7]);

#ifdef __cplusplus
}
#endif

#endif /* CONV_H_ */

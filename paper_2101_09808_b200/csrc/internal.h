// internal.h -- library-internal declarations shared by the host plan code
// and the kernel launchers.  Not part of the ABI (see include/conv.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string>

namespace conv {

// Problem of Eq. 1: H, W are OUTPUT extents.  Stride U,
// dilation D (PAPER.md:201 footnote; Table 1's * layers) and
// zero padding ph, pw: Out[n,k,h,w] sums
// In[n,c,U*h+D*r-ph,U*w+D*s-pw] (zero outside the input); a general plan
// stores its explicit input extents (H = (hin + 2ph - D*(R-1) - 1)/U + 1), a
// plain plan's input is (H+R-1) x (W+S-1).
struct Problem {
    int N, K, C, H, W, R, S;
    int U = 1;              // stride (both axes)
    int hin = 0, win = 0;   // explicit input extents (0: minimal, (H-1)*U + D*(R-1) + 1)
    int D = 1;              // dilation (both axes)
    int ph = 0, pw = 0;     // zero padding rows (top and bottom) / columns (left and right)
    int64_t Hin() const { return hin ? (int64_t)hin : (int64_t)(H - 1) * U + (int64_t)D * (R - 1) + 1 - 2 * ph; }
    int64_t Win() const { return win ? (int64_t)win : (int64_t)(W - 1) * U + (int64_t)D * (S - 1) + 1 - 2 * pw; }
    int64_t rows_span(int h_out) const { return (int64_t)(h_out - 1) * U + (int64_t)D * (R - 1) + 1; }  // input rows of h_out output rows
    int64_t M() const { return (int64_t)N * H * W; }  // implicit-GEMM M
    int64_t in_elems() const { return (int64_t)N * C * Hin() * Win(); }
    int64_t ker_elems() const { return (int64_t)K * C * R * S; }
    int64_t out_elems() const { return (int64_t)N * K * H * W; }
    double flops() const { return 2.0 * (double)N * K * H * W * (double)C * R * S; }
};

// Device facts the selector uses (queried at plan creation).
struct Device {
    int ordinal = 0;
    int sms = 148;
    int cc_major = 10, cc_minor = 0;
    size_t smem_optin = 232448;   // max dynamic smem per block (opt-in)
    size_t l2_bytes = 126u << 20;
    // Bandwidths (bytes/s) and peaks (flop/s) used by the model.  HBM and the
    // bf16 tensor peak default to MEASURED_PEAKS.json's values; the L2->SMEM
    // figure and the FFMA peak are defaults to be replaced by the probes.
    double bw_hbm = 6544.7e9;
    double bw_l2 = 20.0e12;       // L2 -> SMEM via TMA: >= 23 TB/s sustained in the r01
                                  // TMA-only experiment (693 MB in 30 us); 20 TB/s used
    double peak_bf16 = 1651.8e12;
    double peak_tf32 = 825.9e12;
    double peak_fp32 = 74.4e12;
};

// ---- tensor-core path (K3) ------------------------------------------------
struct TcTile {
    int bn = 128;        // GEMM-N tile (output channels), multiple of 32, <= 256
    int stages = 4;      // smem ring depth
    int cg = 1;          // CTAs per MMA: 1 (M = 128) or 2 (CTA pair, M = 256)
    int kbs = 1;         // k-blocks (one TMA box of A and of B each) per pipeline stage
    int fuse = 0;        // 1: the NCHW->NHWC In transform runs inside the main kernel
                         //    (cooperative chunk transform, warps 0-3 of every CTA)
    int tnb = 2;         // fuse: input staging buffers of the transform (2..6)
    int pre_c = 64;      // fuse: channels of wave 0's input converted by the repack launch (prologue)
    int splits = 1;      // split-K (fuse = 0): each tile's k loop in `splits` stage-aligned ranges,
                         //    fp32 partials summed in split order by the tile's last CTA
};

struct TcLayout {        // derived from Problem + element size
    int elem;            // bytes per element in the workspace (4 tf32, 2 bf16)
    int Cp;              // channels padded so that Cp*elem is 32, 64 or a multiple of 128
    int sw;              // swizzle span in bytes = BKc*elem (32, 64 or 128)
    int bkc;             // channels per k-block
    int n_cblk;          // Cp / bkc
    size_t in_ws_bytes;  // NHWC workspace
    size_t ker_ws_bytes; // KRSC workspace
    // cooperative in-kernel transform (fuse = 1): chunks of 64 pixels x cc channels
    int cc;              // channels per chunk: min(32, bkc)
    int nch;             // Cp / cc
    int hh;              // chunks per k-block: bkc / cc
    int64_t npch;        // 64-pixel chunks per input plane
    bool coop_ok;        // TMA-legal NCHW plane (Hin*Win*4 a multiple of 16 B)
    size_t flag_bytes;   // 128 B reserved + one int ready flag per chunk
};
size_t tc_transform_smem_bytes(const TcLayout& L, int tnb);

// Repack launch (repack.cu).  Fused plans (the In transform inside K3):
// besides Ker, the launch clears the chunk flags and converts the
// "prologue" -- channels [0, pre_ch * cc) of input chunk-pixels q < pre_q
// (wave 0's first channel blocks) -- setting those chunks' flags.
struct RepackFuse {
    int* zero_ptr = nullptr;   // 32 reserved ints + the chunk flags [Q][nch]
    int zero_n = 0;
    int pre_q = 0;             // prologue chunk-pixels [0, pre_q)
    int pre_ch = 0;            // channel chunks the prologue covers
    int nch = 0;               // channel chunks per chunk-pixel (flag row length)
    int cc = 0;                // channels per chunk
};
cudaError_t launch_repack(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker,
                          void* in_ws, void* ker_ws, cudaStream_t st, cudaEvent_t* ev, bool with_in,
                          const RepackFuse& fz);

// Tiny-C tap expansion (repack.cu): In' = the R*S*C taps of every output
// pixel as channels ([N][H][W][Cp]), Ker' = [K][Cp] in the same (r, s, c)
// order; the equivalent 1x1 problem is expanded_problem(pb).
cudaError_t launch_expand(const Problem& pb, int Cp, bool bf16, const float* in, const float* ker, void* in_ws,
                          void* ker_ws, cudaStream_t st, cudaEvent_t* ev);
inline Problem expanded_problem(const Problem& pb) {
    Problem pe{pb.N, pb.K, pb.R * pb.S * pb.C, pb.H, pb.W, 1, 1};
    return pe;
}
// Layers for which the expansion pays (the TMA im2col rows would be <= 16 B
// of channels and there are several taps): measured on Table 1's C = 3
// stems (profiles/r01b/expand_ab.jsonl).
inline bool expand_useful(const Problem& pb, bool bf16) {
    const int elem = bf16 ? 2 : 4;
    // the expanded workspace holds R*S*C channels per OUTPUT pixel: bounded
    // at 2 GiB so that large-kernel layers keep the plain im2col path
    return pb.C * elem <= 16 && pb.R * pb.S >= 4 && (int64_t)pb.R * pb.S * pb.C <= 1024 &&
           pb.M() * pb.R * pb.S * pb.C * elem <= ((int64_t)1 << 31);
}

TcLayout tc_layout(const Problem& p, bool bf16);

// Split-K geometry of a tile choice: k iterations per split (stage-aligned)
// and the workspace the partial slabs + arrival counters take (0 if
// t.splits == 1).  A split count whose last range would be empty is invalid
// (tc_split_kper returns 0).
int tc_split_kper(const Problem& pb, const TcLayout& L, const TcTile& t);
size_t tc_split_bytes(const Problem& pb, const TcLayout& L, const TcTile& t);
// Whether a split count is runnable for this tile: fuse = 0, cg = 1, BN <=
// 128, non-empty stage-aligned ranges, the reduction shares fit the pipeline
// smem (the one-wave condition depends on the device: the selector / tc_run).
bool tc_split_ok(const Problem& pb, const TcLayout& L, const TcTile& t);
size_t tc_smem_bytes(const TcLayout& L, const TcTile& t);

// Launch the repack (K1 + K2, one launch) and K3 (tcgen05 implicit GEMM).
// events (optional, n_events == 3) are recorded around each kernel.
// flag_ws: L.flag_bytes of workspace for the fused transform (unused if !t.fuse).
// expand_src (tiny-C plans): p is expanded_problem(*expand_src) and the
// layout transform is the tap expansion of *expand_src (launch_expand).
cudaError_t tc_run(const Problem& p, const TcLayout& L, const TcTile& t, bool bf16,
                   const float* in, const float* ker, float* out, void* in_ws, void* ker_ws, void* flag_ws,
                   cudaStream_t st, int num_sms, cudaEvent_t* ev, std::string& err,
                   const Problem* expand_src = nullptr);

// ---- FP32 SIMT path (K4) ----------------------------------------------------
struct SimtTile {
    int tk = 8;   // output channels per thread (register tile)
    int tw = 4;   // output pixels per thread (stride-32 within a warp)
    int kg = 4;   // channel groups (warps along k) per CTA
    int pw = 2;   // pixel warps per CTA
    int tn = 1;   // images per CTA tile
    int th = 8;   // output rows per image per CTA tile
    int bc = 8;   // input channels per smem stage
    int ver = 1;  // 1: stride-32 pixel slots (any S); 2: consecutive-pixel windows (S in {1,3},
                  //    TW in {4,8}, or TW = W in {7,14}: one thread per output row)
    int splits = 1;   // split-C: CTAs per output tile along C (grid z), partial outputs summed
                      //    in split order by a third kernel (deterministic per split count)
};
size_t simt_smem_bytes(const Problem& p, const SimtTile& t);
size_t simt_ws_bytes(const Problem& p, const SimtTile& t);   // packed Ker (+ split-C partials)
inline int simt_num_kernels(const SimtTile& t) { return t.splits > 1 ? 3 : 2; }
bool simt_v2_ok(const Problem& p);
bool simt_v2_tw_ok(const Problem& p, int tw);
int simt2_pitch(const Problem& p, const SimtTile& t);
bool simt_tile_supported(const SimtTile& t);
// Launch the Ker packing kernel and K4.  events (optional, 3) around each.
cudaError_t simt_run(const Problem& p, const SimtTile& t, const float* in, const float* ker,
                     float* out, void* ws, cudaStream_t st, cudaEvent_t* ev, std::string& err);

// Driver entry points resolved through the runtime (no -lcuda link).
bool driver_init(std::string& err);
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                     cuuint32_t, cuuint32_t, const cuuint32_t*,
                                     CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
extern PFN_encodeTiled g_encode_tiled;
extern PFN_encodeIm2col g_encode_im2col;

}  // namespace conv

// model.cpp -- the tile selector.
//
// The paper's method (MOpt, Sec. 5 and Alg. 1
// PAPER.md:383-419) picks the tiling that minimises the bottleneck level's
// bandwidth-scaled data movement, max_l DV^l / BW^l, subject to per-level
// capacity constraints (Eq. 4).  On a B200 the levels are
// registers/TMEM, shared memory, L2 and HBM; the tile space of each kernel is
// small and discrete, so instead of Ipopt + FloorToInteger + LoadBalancer the
// selector enumerates every feasible candidate and evaluates
//
//   T(cand) = max( FLOPs_issued / peak,  DV_{L2->SMEM} / BW_L2 ) / wave_eff
//             + DV_HBM / BW_HBM (the part not overlapped) + fixed launch costs
//
// where DV_{L2->SMEM} comes from the paper's single-level model (Sec. 3.2,
// conv_model_dv below) instantiated with the CTA tile and the kernel's
// tile-loop order, wave_eff = tiles / (ceil(tiles / slots) * slots) is Sec. 7's
// "prod T/PT == num_cores" load-balance term and DV_HBM counts
// the compulsory traffic plus the layout transforms.
#include <cstdlib>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "../../include/conv.h"
#include "internal.h"
#include "model.h"

// ---------------------------------------------------------------------------
// Sec. 3 / Sec. 2.2 data-movement model (exported: conv_model_*)

namespace {
enum { IN_ = 0, KER_ = 1, OUT_ = 2 };
enum { I_N = 0, I_K = 1, I_C = 2, I_R = 3, I_S = 4, I_H = 5, I_W = 6 };

// Which of the 7 iterators index each tensor (Sec. 4:
// "each of the seven loop indices is present in exactly two of the three
// tensors").
const bool kPresent[3][7] = {
    /* In  [n,c,h+r,w+s] */ {true, false, true, true, true, true, true},
    /* Ker [k,c,r,s]     */ {false, true, true, true, true, false, false},
    /* Out [n,k,h,w]     */ {true, true, false, false, false, true, true},
};

double footprint(int t, const double* T) {
    switch (t) {
        case IN_: return T[I_N] * T[I_C] * (T[I_H] + T[I_R] - 1) * (T[I_W] + T[I_S] - 1);
        case KER_: return T[I_K] * T[I_C] * T[I_R] * T[I_S];
        default: return T[I_N] * T[I_K] * T[I_H] * T[I_W];
    }
}
}  // namespace

extern "C" double conv_model_footprint(const double T[7]) {
    if (!T) return -1;
    return footprint(IN_, T) + footprint(KER_, T) + footprint(OUT_, T);
}

extern "C" double conv_model_dv(const int perm[7], const double Nx[7], const double T[7], double dv[3]) {
    if (!perm || !Nx || !T) return -1;
    bool seen[7] = {false};
    for (int i = 0; i < 7; ++i) {
        if (perm[i] < 0 || perm[i] > 6 || seen[perm[i]]) return -1;
        seen[perm[i]] = true;
        if (!(T[i] >= 1) || !(Nx[i] >= 1) || T[i] > Nx[i]) return -1;
    }
    double trip[7];
    for (int d = 0; d < 7; ++d) trip[d] = ceil(Nx[d] / T[d]);
    double out[3];
    for (int t = 0; t < 3; ++t) {
        // R_A: innermost tile loop whose iterator indexes A (perm[6] is innermost).
        int ra = -1;
        for (int i = 6; i >= 0; --i)
            if (kPresent[t][perm[i]]) { ra = i; break; }
        const int it = perm[ra];
        if (t == IN_ && (it == I_W || it == I_H || it == I_S || it == I_R)) {
            // Case 2: partial reuse along the innermost
            // present iterator; loops strictly outside it multiply.
            double outer = 1;
            for (int i = 0; i < ra; ++i) outer *= trip[perm[i]];
            double partial;
            const double spanh = T[I_H] + T[I_R] - 1, spanw = T[I_W] + T[I_S] - 1;
            const double base = T[I_N] * T[I_C];
            switch (it) {
                case I_W: partial = base * spanh * T[I_W] * (trip[I_W] - 1); break;
                case I_S: partial = base * spanh * T[I_S] * (trip[I_S] - 1); break;
                case I_H: partial = base * T[I_H] * (trip[I_H] - 1) * spanw; break;
                default:  partial = base * T[I_R] * (trip[I_R] - 1) * spanw; break;
            }
            out[t] = outer * (footprint(IN_, T) + partial);
        } else {
            // Case 1: a fresh slice every time the
            // iterator at R_A (or any loop outside it) changes.
            double cnt = 1;
            for (int i = 0; i <= ra; ++i) cnt *= trip[perm[i]];
            out[t] = cnt * footprint(t, T) * (t == OUT_ ? 2.0 : 1.0);
        }
    }
    if (dv) { dv[0] = out[0]; dv[1] = out[1]; dv[2] = out[2]; }
    return out[0] + out[1] + out[2];
}

extern "C" double conv_model_dv_matmul(const int perm[3], const double Nx[3], const double T[3]) {
    // Sec. 2.2: C[i][j] += A[i][k] * B[k][j]; same two-case
    // rule with index sets A{i,k}, B{k,j}, C{i,j} (C read + written: x2).
    if (!perm || !Nx || !T) return -1;
    static const bool pres[3][3] = {{true, false, true}, {false, true, true}, {true, true, false}};
    bool seen[3] = {false};
    for (int i = 0; i < 3; ++i) {
        if (perm[i] < 0 || perm[i] > 2 || seen[perm[i]]) return -1;
        seen[perm[i]] = true;
        if (!(T[i] >= 1) || T[i] > Nx[i]) return -1;
    }
    double trip[3];
    for (int d = 0; d < 3; ++d) trip[d] = ceil(Nx[d] / T[d]);
    const double fp[3] = {T[0] * T[2], T[2] * T[1], T[0] * T[1]};
    double total = 0;
    for (int a = 0; a < 3; ++a) {
        int ra = -1;
        for (int i = 2; i >= 0; --i)
            if (pres[a][perm[i]]) { ra = i; break; }
        double cnt = 1;
        for (int i = 0; i <= ra; ++i) cnt *= trip[perm[i]];
        total += cnt * fp[a] * (a == 2 ? 2.0 : 1.0);
    }
    return total;
}

// ---------------------------------------------------------------------------
// Selector

namespace conv {

static const double kLaunchUs = 2.0;      // per-kernel launch + ramp
// halo kernel (single launch): fixed per-CTA chain (barrier init, TMEM
// alloc, Ker conversion, MMA issue), staged-input bandwidth per SM and the
// epilogue's store bandwidth per SM -- first estimates, r02
static const double kHaloFixedUs = 1.5;
static const double kHaloBW = 60e9;
static const double kHaloEpiBW = 40e9;
static const double kTileOverheadUs = 0.25;  // per wave: pipeline fill + epilogue drain

static double wave_eff(long tiles, long slots) {
    if (tiles <= 0 || slots <= 0) return 1.0;
    const long waves = (tiles + slots - 1) / slots;
    return (double)tiles / (double)(waves * slots);
}

// GPU instantiation of the Sec. 3.2 model for the implicit GEMM's CTA tile:
// pixels are one flattened dimension (T_w = 128 of N_w = M), T_k = BN,
// T_c = BKc, T_r = T_s = 1; tile-loop order (outer -> inner) = pixel tile,
// k tile, r, s, c-block.  In and Ker are case 1 (innermost ct), i.e. the
// im2col replay; Out leaves the SM from TMEM straight to global, so only
// In + Ker cross L2 -> SMEM.
static double tc_dv_l2_smem_bytes(const Problem& pb, const TcLayout& L, int bn, int cg) {
    const int perm[7] = {I_N, I_H, I_W, I_K, I_R, I_S, I_C};
    const double Nx[7] = {1, (double)pb.K, (double)L.Cp, (double)pb.R, (double)pb.S, 1, (double)pb.M()};
    const double T[7] = {1, (double)std::min(bn, pb.K), (double)L.bkc, 1, 1, 1,
                         (double)std::min<int64_t>(128 * cg, pb.M())};
    double dv[3];
    conv_model_dv(perm, Nx, T, dv);
    // Trip counts are ceil(N/T): partial tiles are charged as full tiles
    // (TMA moves whole boxes; out-of-bounds rows are zero-filled, not read).
    return (dv[IN_] + dv[KER_]) * L.elem;
}

// Shared-memory port of one SM (128 B/clk): the TMA writes every operand byte
// once and the tensor core reads it once.  The pair's B half is read by its
// own SM only, so per SM per k-block: 2 * (128 + BN/cg) * sw bytes.
static const double kSmemBytesPerClk = 128.0;
static const double kClockHz = 1.84e9;   // SM clock measured under tcgen05 load (scripts/probe_mma.cu)
// tcgen05.mma issue model (measured, scripts/probe_mma.cu and the r01
// timeline trace): one 128 x N x 32-byte-K MMA takes max(N/2, 48) cycles on
// an SM; every pipeline stage adds ~150 cycles of barrier / commit bubble.
static const double kStageBubbleClk = 150.0;
static const double kStageLatClk = 800.0;
static const double kEpiStoreBW = 5.0e12;  // bytes/s the whole chip's epilogues drain at
// fused transform (measured r01b, batched layer): 67 MB of fp32 In in ~35 us
// per 148 CTAs while the MMAs run, 9% MMA slowdown, ~6 us startup chain
static const double kTransformBW = 1.9e12;
// Split-K epilogue: arrival fence + atomic + wait + the share's bulk copy
// round trip, and one SM's L2 read rate for the reduction share.  Fitted to
// the r01b Table-1 A/B (profiles/r01b/splitk_ab.jsonl): with 2.5 us the
// modeled gain of every split layer matches the measured one within ~1 us,
// and the shallow-k layers (R6, R7, M4: 18 k-blocks), where splitting
// measured 1-2 us slower, stay unsplit.
static const double kSplitSyncUs = 2.5;
static const double kSplitReadBW = 150e9;
static const double kTransformDrag = 1.09;
static const double kTransformStartUs = 6.0;

ModelResult model_tc(const Problem& pb, const Device& dev, bool bf16, const TcTile& t) {
    ModelResult r;
    const TcLayout L = tc_layout(pb, bf16);
    const long tm = 128L * t.cg;
    const long mt = (long)((pb.M() + tm - 1) / tm), nt = (pb.K + t.bn - 1) / t.bn;
    const long units = dev.sms / t.cg;
    const int splits = std::max(1, t.splits);
    r.tiles = mt * nt;
    const long work = r.tiles * splits;                 // split-K work items
    r.ctas = std::min<long>(work, units) * t.cg;
    r.wave_eff = wave_eff(work, units);
    const double peak = bf16 ? dev.peak_bf16 : dev.peak_tf32;
    const double flops_issued = 2.0 * (double)mt * tm * (double)nt * t.bn * (double)pb.R * pb.S * L.Cp;
    r.t_comp_us = flops_issued / peak * 1e6;
    r.dv_l2_smem = tc_dv_l2_smem_bytes(pb, L, t.bn, t.cg);
    r.t_l2_us = r.dv_l2_smem / dev.bw_l2 * 1e6;
    // tensor pipe of the busiest unit: ceil(tiles/units) tiles, each
    // R*S*n_cblk/kbs stages of kbs*(sw/32) MMAs.
    const double tiles_per_unit = ceil((double)work / units);
    const double stages_per_tile = (double)tc_split_kper(pb, L, t) / t.kbs;   // per work item
    const double mma_clk = std::max(t.bn / 2.0, 48.0);
    // a stage also cannot turn over faster than the producer -> TMA -> MMA
    // -> commit round trip allows (kStageLatClk, r01b selector study: on
    // long-K few-tile layers time scales with the number of stages)
    const double stage_clk = std::max(t.kbs * (L.sw / 32.0) * mma_clk + kStageBubbleClk, kStageLatClk);
    const double t_pipe_us = tiles_per_unit * stages_per_tile * stage_clk / kClockHz * 1e6;
    const double kblocks_per_sm = (double)r.tiles * pb.R * pb.S * L.n_cblk / units;
    const double t_smem_us = kblocks_per_sm * 2.0 * (128.0 + (double)t.bn / t.cg) * L.sw /
                             kSmemBytesPerClk / kClockHz * 1e6;
    // last tile's epilogue is not overlapped: every CTA stores 128 x BN fp32
    double t_tail_us = std::min<double>(work * t.cg, dev.sms) * 128.0 * std::min(t.bn, pb.K) * 4.0 / kEpiStoreBW * 1e6;
    if (splits > 1) {
        // partial slab store + arrival (fence, atomic, wait for the tile's
        // other splits) + each CTA's reduction share: the tile's `splits`
        // slabs over 1/splits of the columns = one slab's bytes per CTA from
        // L2 (~kSplitReadBW per SM)
        t_tail_us = 2.0 * t_tail_us + kSplitSyncUs + 128.0 * t.bn * 4.0 / kSplitReadBW * 1e6;
    }
    // HBM: repacks (read fp32 In/Ker, write workspace) + main kernel (read
    // workspace once -- the 9x im2col replay and the k-tile re-reads hit L2 --
    // and write fp32 Out once).
    const double repack = 4.0 * pb.in_elems() + (double)L.in_ws_bytes + 4.0 * pb.ker_elems() + (double)L.ker_ws_bytes;
    const double main_hbm = (double)L.in_ws_bytes + (double)L.ker_ws_bytes + 4.0 * pb.out_elems();
    r.dv_hbm = repack + main_hbm;
    r.t_hbm_us = r.dv_hbm / dev.bw_hbm * 1e6;
    // (t_comp_us, at the MEASURED_PEAKS cuBLAS rate, is reported only: the
    // tensor pipe term t_pipe uses the measured per-MMA cycle counts.)
    const double t_main = std::max({t_pipe_us, r.t_l2_us / r.wave_eff,
                                    t_smem_us / r.wave_eff, main_hbm / dev.bw_hbm * 1e6})
                          + t_tail_us + kLaunchUs;
    double t_rep = repack / (0.8 * dev.bw_hbm) * 1e6 + 2 * kLaunchUs;
    double t_main_f = t_main;
    if (t.fuse) {
        // Cooperative In transform inside the main kernel (measured r01b,
        // profiles/r01b/fuse_sweep.log): the repack launch converts only the
        // prologue (pre_c channels of wave 0's input) besides Ker; the rest of
        // In is converted by every CTA's transform warps at ~kTransformBW,
        // overlapped with the MMAs but slowing them by kTransformDrag (they
        // share the SM's shared-memory port, L2 and issue slots).  While the
        // transform has not caught up, wave 0 waits: the part of its input
        // beyond the prologue must be converted before its last channel
        // block can run.  Every fused plan also pays the chunk pipeline's
        // startup chain (decode, load, convert, store, publish, watch):
        // charged to single-wave layers only, the model picked the fused
        // transform for the large-M batch-1 Table-1 layers Y0/Y2/Y5, where it
        // measured 2-8 us slower than the separate repack (r01b
        // profiles/r01b/selector_fuse.jsonl); only the batched layer gains.
        const double in_rd = 4.0 * pb.in_elems();
        const double waves = ceil((double)r.tiles / units);
        const double pre_frac = std::min(1.0, (double)t.pre_c / L.Cp) / std::max(1.0, waves);
        const double t_tr = in_rd * (1.0 - pre_frac) / kTransformBW * 1e6;
        const double wave0_in = in_rd / std::max(1.0, waves) * (1.0 - std::min(1.0, (double)t.pre_c / L.Cp));
        const double stall0 = std::max(0.0, wave0_in / kTransformBW * 1e6 - t_pipe_us / std::max(1.0, waves));
        t_main_f = std::max(t_main * kTransformDrag, t_tr) + stall0 + kTransformStartUs;
        const double pre_bytes = (4.0 + L.elem) * pb.in_elems() * pre_frac;
        t_rep = (4.0 * pb.ker_elems() + (double)L.ker_ws_bytes + pre_bytes) / (0.8 * dev.bw_hbm) * 1e6 + 2 * kLaunchUs;
        r.dv_hbm = in_rd + (double)L.in_ws_bytes + 4.0 * pb.ker_elems() + 2.0 * (double)L.ker_ws_bytes + 4.0 * pb.out_elems();
        r.t_hbm_us = r.dv_hbm / dev.bw_hbm * 1e6;
    }
    r.model_us = t_main_f + t_rep;
    r.smem = tc_smem_bytes(L, t);
    return r;
}

static int tc_max_stages(const Device& dev, const TcLayout& L, int bn, int cg, int kbs, int fuse) {
    for (int s = 8; s >= 2; --s) {
        TcTile t;
        t.bn = bn;
        t.stages = s;
        t.cg = cg;
        t.kbs = kbs;
        t.fuse = fuse;
        t.tnb = 2;
        if (tc_smem_bytes(L, t) <= dev.smem_optin) return s;
    }
    return 0;
}

bool select_tc(const Problem& pb, const Device& dev, bool bf16, TcTile& best, ModelResult& best_r, const TcForce& f,
               std::string& why) {
    const int force_bn = f.bn, force_stages = f.stages, force_cg = f.cg, force_kbs = f.kbs, force_fuse = f.fuse,
              force_pre_c = f.pre_c;
    const TcLayout L = tc_layout(pb, bf16);
    {
        // the TMA im2col bounding-box corners of a 4-D map lie in [-128, 127]:
        // lower = -pad, upper = pad - D*(R-1)
        const int64_t uh = pb.ph - (int64_t)pb.D * (pb.R - 1), uw = pb.pw - (int64_t)pb.D * (pb.S - 1);
        if (pb.ph > 128 || pb.pw > 128 || uh < -128 || uw < -128 || uh > 127 || uw > 127) {
            why = "pad > 128 or pad - D*(R-1) outside [-128, 127]: the TMA im2col bounding box of a 4-D map is limited";
            return false;
        }
    }
    if (pb.U > 8) { why = "stride > 8: the TMA im2col traversal stride is limited to 8"; return false; }
    if (pb.M() + 256 > (int64_t)INT32_MAX) { why = "N*H*W too large for the tensor path"; return false; }
    if (force_fuse == 1 && !L.coop_ok) {
        why = "fuse=1 needs (H+R-1)*(W+S-1) % 4 == 0 (TMA-legal NCHW plane)";
        return false;
    }
    static const int kBNs[] = {32, 64, 128, 192, 256};
    bool found = false;
    for (int cg = 1; cg <= 2; ++cg) {
        if (force_cg && cg != force_cg) continue;
        // k-blocks per stage; must divide the k loop.  7 and 9 are whole
        // kernel rows / windows of 7x7 and 3x3 taps: tiny-C layers (C*elem
        // <= 128 B: one k-block per tap) otherwise pay the per-stage latency
        // floor once per tap (R1: 49 stages of 16 channels per tile).
        for (int kbs : {1, 2, 3, 4, 6, 7, 8, 9}) {
            if (force_kbs && kbs != force_kbs) continue;
            if ((pb.R * pb.S * L.n_cblk) % kbs) continue;
            for (int bn : kBNs) {
                if (force_bn && bn != force_bn) continue;
                if (f.bn_max && bn > f.bn_max) continue;
                if (!force_bn && bn > 32 && bn / 2 >= pb.K) continue;   // mostly padding
                // CTA pairs halve the B operand traffic, which is negligible at
                // BN = 32, while their cluster synchronisation lengthens a
                // latency-bound k-loop: measured r01b on Table-1 M9 (M = 25,
                // C*R*S = 9216) 92 us paired vs 53 us single at BN = 32
                if (cg == 2 && bn < 64 && !force_cg) continue;
                for (int fuse = 0; fuse <= 1; ++fuse) {
                    if (force_fuse >= 0 ? fuse != force_fuse : (fuse && !L.coop_ok)) continue;
                    const int smax = tc_max_stages(dev, L, bn, cg, kbs, fuse);
                    // at least 4 k-blocks in flight (3 stages of 1-2 k-blocks, 2 of
                    // 4) unless forced: fewer cannot overlap loads and MMAs well.
                    // (r01b selector study: kbs = 4 x 2 stages is the measured
                    // best on the tiny-M Table-1 layers M7, M9, R12, Y12.)
                    if (smax < (force_stages || force_kbs ? 2 : (kbs >= 4 ? 2 : 3))) continue;
                    TcTile t;
                    t.bn = bn;
                    t.cg = cg;
                    t.kbs = kbs;
                    t.fuse = fuse;
                    t.stages = force_stages ? force_stages : smax;
                    if (t.stages < 2 || t.stages > smax) continue;
                    if (fuse) {   // as many transform chunk buffers as fit (2..6)
                        // prologue depth measured best in r01b (batched layer, after the
                        // production-build cleanup): 192 channels bf16 (915-917 vs 905-906
                        // TFLOP/s at 128), 64 tf32 (603.5 vs 589-597 at 96-192)
                        t.pre_c = force_pre_c >= 0 ? force_pre_c : (bf16 ? 192 : 64);
                        t.tnb = 2;
                        for (int nb = 6; nb > 2; --nb) {
                            TcTile u = t;
                            u.tnb = nb;
                            if (tc_smem_bytes(L, u) <= dev.smem_optin) { t.tnb = nb; break; }
                        }
                    }
                    // split-K (not fused): only while the tiles do not fill one
                    // wave -- the k loop of a few long tiles then spreads over
                    // the idle SMs (PAPER.md:375 parallelises over output
                    // dimensions only: 8 CPU cores; 148 SMs at batch 1 need
                    // the reduction split)
                    const long tiles = ((pb.M() + 128L * cg - 1) / (128L * cg)) * ((pb.K + bn - 1) / bn);
                    const long units = dev.sms / cg;
                    static const int kFree[] = {1, 2, 3, 4, 6, 8, 12, 16};
                    const int forced[] = {f.splits};
                    const int* cand = f.splits ? forced : kFree;
                    const int ncand = f.splits ? 1 : 8;
                    for (int ci = 0; ci < ncand; ++ci) {
                        const int sp = cand[ci];
                        // (one wave: the split CTAs of a tile wait for each other)
                        if (sp > 1 && (fuse || tiles * sp > units)) continue;
                        t.splits = sp;
                        if (!tc_split_ok(pb, L, t)) continue;
                        ModelResult r = model_tc(pb, dev, bf16, t);
                        if (!found || r.model_us < best_r.model_us) { best = t; best_r = r; found = true; }
                    }
                }
            }
        }
    }
    // the single-launch halo kernel (halo.cu): one CTA per 128-pixel tile of
    // the padded grid, the whole layer in one launch -- modeled as launch +
    // the per-CTA chain (staged input at ~kHaloBW per SM, the R*S*rowb/32
    // MMAs, the 128 x K fp32 epilogue) per wave
    // Only on request (tile key halo=1): measured r02 (profiles/r02/
    // bench_small_halo_*.jsonl) it does not beat the two-launch im2col plans
    // on the BASELINE layers (det 14.4 vs 13.8 us, r2 14.4 vs 12.0, pw 18.4 vs
    // 10.3, tiny 10.4 vs 10.4): the per-CTA chain -- cold input copy 2.3 us,
    // conversion 0.9, dependent MMAs 1.7, epilogue 1.7 -- is not shorter
    // than the im2col kernel's, and the protocol floor of one launch is 6 us.
    const bool halo_forced = f.halo == 1;
    if (halo_forced && halo_ok(pb, bf16, dev.smem_optin) && !f.bn && !f.cg && !f.kbs && f.splits <= 1 &&
        f.fuse != 1) {
        ModelResult r;
        const int64_t ctas = halo_ctas(pb);
        const double waves = ceil((double)ctas / dev.sms);
        const double stage_bytes = 4.0 * pb.C * (128.0 + (pb.R - 1) * (double)pb.Win() + pb.S - 1);
        const double epi_bytes = 128.0 * pb.K * 4.0;
        const double per_cta_us = kHaloFixedUs + stage_bytes / kHaloBW * 1e6 + epi_bytes / kHaloEpiBW * 1e6;
        r.tiles = (long)ctas;
        r.ctas = (long)std::min<int64_t>(ctas, dev.sms);
        r.wave_eff = (double)ctas / (waves * dev.sms);
        const double flops_issued = 2.0 * (double)ctas * 128.0 * pb.K * pb.R * pb.S * pb.C;
        r.t_comp_us = flops_issued / (bf16 ? dev.peak_bf16 : dev.peak_tf32) * 1e6;
        r.dv_l2_smem = (double)ctas * (stage_bytes + 4.0 * pb.ker_elems());
        r.t_l2_us = r.dv_l2_smem / dev.bw_l2 * 1e6;
        r.dv_hbm = 4.0 * (pb.in_elems() + pb.ker_elems() + pb.out_elems());
        r.t_hbm_us = r.dv_hbm / dev.bw_hbm * 1e6;
        r.model_us = kLaunchUs + std::max({waves * per_cta_us, r.t_hbm_us, r.t_l2_us});
        r.smem = 0;
        if (halo_forced || !found || r.model_us < best_r.model_us) {
            best = TcTile();
            best.halo = 1;
            best.bn = pb.K;
            best.stages = 1;
            best_r = r;
            found = true;
        }
    } else if (halo_forced) {
        why = "layer not eligible for the halo kernel (stride/dilation/padding 1/1/0, C*elem <= 128 B, K <= 256, "
              "smem) or other tile keys forced";
        return false;
    }
    if (!found) why = "no tensor-path tile fits shared memory / TMEM for this request";
    return found;
}

// ---- SIMT -------------------------------------------------------------------
// Issue cost per element of the v2 per-row 4-B copy loop (taken when the
// 16-B copy plan does not fit 4 units per thread).  r01b: 24 from the batched
// layer (~2.3x slower layer); the Table-1 study (simt_study2: Y18 bc 4 -> 8
// crossed into it, 2.78 -> 8.07 us per chunk) measured ~3x more.
static const double kSimtSlowCopy = 72.0;
// The same loop with 16-B copies (rows 16-B aligned, Win % 4 == 0; r01b):
// the Table-1 AUTO sweep with 24 vs 72 (two runs each, profiles/r01b/
// t1_simt_slowcopy16.jsonl) 2695 -> 2681 us (Y0 57.4 -> 47.1, Y2, Y4 -4 %;
// R7 +8 %, Y5 +3 %).
static const double kSimtSlowCopy16 = 24.0;
// (env CONV_SIMT_CHUNK_SYNC overrides it: the selector study of this term)
static const double kSimtChunkSyncClk = [] {
    const char* e = getenv("CONV_SIMT_CHUNK_SYNC");
    return e ? atof(e) : 0.0;
}();

// Registers per thread of the kernel instance a tile launches (simt.cu
// dispatch_simt2 / dispatch_simt), as ptxas allocated them in the built
// library (simt_regs.inc, scripts/gen_simt_regs.py; tests/test_abi.py checks
// it against libconv.so).  The former estimate (TK*TW + TK + window + 24 for
// v2) said 72 for v2 TK=8 TW=4 S=3 where ptxas gives 104-128: 2 CTAs per SM
// modeled where 1 fits (ncu r01b Y0: occupancy limited by registers to 1).
struct SimtRegs { int ver, tk, tw, kr, ks, splitc, tma, regs; };
static const SimtRegs kSimtRegs[] = {
#include "simt_regs.inc"
};

static int simt_regs(const Problem& pb, const SimtTile& t, int win) {
    const int sc = t.splits > 1 ? 1 : 0;
    const int kr = (t.ver == 2 && pb.R == pb.S && (pb.S == 1 || pb.S == 3)) ? pb.R : 0;
    const int ks = t.ver == 2 ? pb.S : 0;
    const int tma = t.ver == 2 && simt2_layout(pb, t).tma ? 1 : 0;
    for (const SimtRegs& e : kSimtRegs)
        if (e.ver == t.ver && e.tk == t.tk && e.tw == t.tw && e.kr == kr && e.ks == ks && e.splitc == sc &&
            e.tma == tma)
            return e.regs;
    // an instance the table does not list (not built): the old estimate
    return std::min(128, t.tk * t.tw + t.tk + win + (t.ver == 2 ? 24 : 2 * t.tw + 28));
}

ModelResult model_simt(const Problem& pb, const Device& dev, const SimtTile& t) {
    ModelResult r;
    const int bko = t.kg * t.tk;
    const long ntile = (pb.N + t.tn - 1) / t.tn, htile = (pb.H + t.th - 1) / t.th, ktile = (pb.K + bko - 1) / bko;
    const double nchunks_all = ceil((double)pb.C / t.bc);
    const int splits = std::max(1, std::min(t.splits, (int)nchunks_all));
    r.tiles = t.flat ? (long)simt_ctas(pb, t, pb.N)   // flat: 32*pw (image, row) slots per CTA
                     : ntile * htile * ktile * splits;  // CTAs (split-C: one per split of a tile)
    const int threads = 32 * t.kg * t.pw;
    const size_t smem = simt_smem_bytes(pb, t);
    r.smem = smem;
    if (smem == SIZE_MAX) { r.model_us = 1e30; return r; }
    // Register level (Sec. 6 microkernel analog): TK*TW accumulators + the
    // input window + TK kernel values + addressing; ptxas caps at 128.
    const int win = t.ver == 2 ? (t.tw + pb.S - 1 + 3) / 4 * 4 : t.tw;
    const int regs = simt_regs(pb, t, win);
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * threads);
    const int by_smem = (int)(228 * 1024 / (smem + 1024));
    const int by_thr = 2048 / threads;
    const int per_sm = std::min({by_regs, by_smem, by_thr, 32});
    if (per_sm < 1) { r.model_us = 1e30; return r; }
    // CTAs land round-robin on the SMs: the busiest SM runs ceil(tiles/SMs)
    // of them, `conc` at a time.
    // (remainder launch, simt_rem_tiles: the busiest SM runs one CTA less and
    // one remainder warp, 1 / kg of a CTA's issue, beside its resident CTAs)
    const int rem = simt_rem_tiles(pb, t, dev.sms);
    const long per_sm_total = (r.tiles + dev.sms - 1) / dev.sms - (rem > 0 ? 1 : 0);
    const long conc = std::min<long>(per_sm, per_sm_total);
    const long waves = (per_sm_total + conc - 1) / conc;
    r.ctas = std::min<long>(r.tiles, (long)per_sm * dev.sms);
    r.wave_eff = (double)r.tiles / ((double)dev.sms * per_sm_total);
    // FFMA issue: 128 lanes/clk/SM at >= 8 resident warps (2 per SMSP hide
    // the LDS latency), proportionally less below.  Per (c, r) the register
    // tile costs: v1 S*(TW + TK/4 + 1) loads/address ops, v2 WIN/4 + S*TK/4 + 3.
    // ncu r01: 8 resident warps/SM issue on only ~54% of cycles; more are
    // needed to cover the LDS/FFMA dependency latencies (12, fitted below).
    const double warps = (double)conc * threads / 32.0;
    // one resident CTA per SM cannot hide its own chunk barriers / copy
    // waits behind another CTA's FFMAs (measured r01b: 512-thread row-mode
    // tiles 1501 us vs 2 x 256-thread tiles 1321 us, same warps per SM)
    // Re-fitted once the model had the real registers per instance (r01b,
    // Table-1 AUTO sweep, profiles/r01b/t1_simt_occupancy.jsonl): 12 warps
    // and 0.7 vs the former 16 and 0.88: 2675 -> 2649 us (R1 -12 %, M3 / M5 /
    // M6 -9..-11 %; Y2 +4 %); the batched layer's tile is unchanged.
    // (v2 runs FFMA2 since r02b, which occupies the FMA pipe two cycles per
    // instruction, so fewer warps keep it busy; env CONV_SIMT_EFF_WARPS /
    // CONV_SIMT_EFF_LONE: the v2 occupancy study, defaults = the r01b fit)
    static const double eff_warps = getenv("CONV_SIMT_EFF_WARPS") ? atof(getenv("CONV_SIMT_EFF_WARPS")) : 12.0;
    static const double eff_lone = getenv("CONV_SIMT_EFF_LONE") ? atof(getenv("CONV_SIMT_EFF_LONE")) : 0.7;
    const double eff = t.ver == 2 ? std::min(1.0, warps / eff_warps) * (conc == 1 ? eff_lone : 1.0)
                                  : std::min(1.0, warps / 12.0) * (conc == 1 ? 0.7 : 1.0);
    const double fma_cr = (double)pb.S * t.tk * t.tw;
    const double over_cr = t.ver == 2 ? win / 4.0 + pb.S * t.tk / 4.0 + 3.0
                                      : pb.S * (t.tw + t.tk / 4.0 + 1.0);
    // v2 with several pixel groups per row (TW = 4 / 8) measured ~1.25x its
    // modeled issue cost relative to row mode (TW = W, one group per row:
    // aligned windows, no padded pixels) on the batched layer (r01b,
    // scripts/simt_sweep3.py: 1571 vs 1321 us against models 1100 / 1152).
    const bool row_mode = t.ver == 2 && (pb.W + t.tw - 1) / t.tw == 1;
    // v1 (strided scalar loads) measured 3.5x its model on r2 (62.5 vs 17.8
    // us, r01b simt_sweep2): charged 4x so that it is picked only where v2
    // cannot run (S not in {1, 3})
    // Flat row-mode tiles (every lane an output row) measured ~4 % slower per
    // CTA than per-image row tiles of the same register tile (r02c,
    // profiles/r02c/flat_ab.txt: (T - 35 us) / (CTAs per SM) = 86.8-87.6 vs
    // 83.5-84.3 us on the batched layer at N = 256 / 128 -- the box's zero
    // rows up to rows_box and the 4-channel chunks their smem allows)
    static const double kSimtFlatCost = 1.04;
    const double issue_factor = (1.0 + over_cr / fma_cr) * (t.ver == 2 ? (row_mode ? 1.0 : 1.25) : 4.0) *
                                (t.flat ? kSimtFlatCost : 1.0);
    const double chunks = ceil(nchunks_all / splits);    // per CTA
    // one chunk: every thread's FFMAs, plus the cp.async copies (one per 4-B
    // element in v1/v2 In rows, ~6 instructions each, spread over the CTA)
    const double fma_chunk_cta = (double)threads * t.tk * t.tw * t.bc * pb.R * pb.S * issue_factor;
    const double in_elems_chunk = (double)t.bc * t.tn * pb.rows_span(t.th) * (pb.Win() + 2 * pb.pw);
    // v2 copies 16-B units from a per-thread plan when they fit 4 per thread;
    // beyond that a per-row loop of 4-B copies runs (~2.3x slower layer
    // measured r01b)
    const double units_v2 = (double)t.bc * t.tn * pb.rows_span(t.th) * (pb.Win() % 4 == 0 ? pb.Win() / 4.0 : pb.Win());
    const double copy_unit = (t.ver == 2 && units_v2 > 4.0 * threads)
                                 ? (pb.Win() % 4 == 0 ? kSimtSlowCopy16 : kSimtSlowCopy) : 6.0;
    // TMA layout (simt2_layout): one thread issues the In box and the Ker
    // bulk copy; the other threads only pass the barrier and the mbarrier
    // wait (~20 issue slots per warp per chunk; lane-instructions here)
    const bool tma = t.ver == 2 && simt2_layout(pb, t).tma;
    const double copy_chunk_cta = tma ? 20.0 * threads + 100.0 * 32.0
                                      : in_elems_chunk * copy_unit + (double)t.bc * pb.R * pb.S * bko / 4.0 * 6.0;
    const double clk = dev.peak_fp32 / (dev.sms * 256.0);      // Hz implied by the FP32 peak
    // a chunk cannot take less than one L2 round trip + two barriers
    const double issue_cyc = (double)conc * (fma_chunk_cta + copy_chunk_cta) / (128.0 * eff);
    // (+ a per-chunk synchronisation charge: a study knob, default 0 --
    // see the bc tie-break in select_simt)
    // Flat tiles are charged ~400 clk per chunk round (r02e, profiles/r02e/bc6/: on the kg = 8 flat
    // tile 6-channel chunks -- 43 ring waits / barriers per CTA instead of 64 -- run 1074 vs 1088 us at
    // N = 256, 567 vs 574 at N = 128, 319 vs 321 at N = 64: 14 us / (3 CTA rounds x 21 chunks) ~ 440 clk)
    static const double kSimtFlatChunkSyncClk = getenv("CONV_SIMT_FLAT_SYNC") ? atof(getenv("CONV_SIMT_FLAT_SYNC")) : 400.0;
    const double chunk_cyc = std::max(issue_cyc, 2000.0) + kSimtChunkSyncClk + (t.flat ? kSimtFlatChunkSyncClk : 0.0);
    // v2 (FFMA2): the time goes with the CTAs each SM runs, not with whole
    // waves -- measured r02b (profiles/r02b/e2e/simt_time_vs_batch.txt,
    // shard_tiles.txt): the batched tile at N = 6..256 takes 35 + 85 k us for
    // k = ceil(CTAs / SMs), and at N = 128 the 7-CTA-per-SM kg = 4 tile beat
    // the 3.5-wave kg = 8 one that whole-wave counting preferred (621 vs
    // 698 us); a finished CTA's slot is refilled at once, so the last wave
    // costs its share.  (CONV_SIMT_WHOLE_WAVES=1: the r01b whole-wave count.)
    static const bool whole_waves = getenv("CONV_SIMT_WHOLE_WAVES") != nullptr;
    const double wv = ((t.ver == 2 && !whole_waves) ? (double)per_sm_total / (double)conc : (double)waves) +
                      (rem > 0 ? 1.0 / (t.kg * (double)conc) : 0.0);
    r.issue_cyc = wv * chunks * issue_cyc;
    r.t_comp_us = wv * chunks * chunk_cyc / clk * 1e6;
    // L2 -> SMEM: per CTA, every c-chunk loads the In halo tile and Ker slab
    // (Eq. 4's In and Ker footprints).
    const double ker_stage = (double)t.bc * pb.R * pb.S * bko;
    r.dv_l2_smem = (double)r.tiles * chunks * (in_elems_chunk + ker_stage) * 4.0;
    r.t_l2_us = r.dv_l2_smem / dev.bw_l2 * 1e6;
    r.dv_hbm = 4.0 * (pb.in_elems() + 2.0 * pb.ker_elems() + pb.out_elems());
    r.t_hbm_us = r.dv_hbm / dev.bw_hbm * 1e6;
    r.model_us = std::max({r.t_comp_us, r.t_l2_us / r.wave_eff, r.t_hbm_us}) + 2 * kLaunchUs;
    if (splits > 1)   // the reduce kernel: a launch + S partial outputs read, Out written
        r.model_us += kLaunchUs + (splits + 1.0) * 4.0 * pb.out_elems() / dev.bw_hbm * 1e6;
    return r;
}

bool select_simt(const Problem& pb, const Device& dev, SimtTile& best, ModelResult& best_r,
                 const SimtTile* forced, unsigned forced_mask, std::string& why) {
    bool found = false;
    const int tks[2] = {4, 8};
    const int kgs[4] = {1, 2, 4, 8};   // (3, 5, 6: CTAs of 3-6 warps load the 4 SMSPs unevenly; flat r02c 1.2-1.3x slower)
    const int bcs[6] = {2, 4, 8, 16, 6, 12};   // 2, 12 (and 6 on other than flat tiles): forced only
    const int tn_max = std::min(pb.N, 16);
    // v2 first when it can run and nothing is forced; v1 only if no v2 tile fits
    const bool tile_forced = forced && (forced_mask & ~(256u | 1024u));   // a tile key other than splits / rem
    const bool v2_first = simt_v2_ok(pb) && !tile_forced;
    const int vers[2] = {v2_first ? 2 : 1, v2_first ? 1 : 2};
    for (int ver : vers) {
    if (ver == 2 && !simt_v2_ok(pb)) continue;
    if (forced && (forced_mask & 128) && ver != forced->ver) continue;
    // v1 only where v2 cannot run (S not in {1, 3}, stride, dilation,
    // padding) unless forced: on every layer measured where both run, the
    // best v2 tile beat the best v1 tile (r01b profiles/r01b/simt_study2.jsonl:
    // Y19 139 vs 450 us, Y13 74 vs 256, Y18 356 vs 430), while the model
    // ranked v1 first on the 1x1 layers (modeled 69 us, measured 471)
    // (automatic selection only: forced keys may name a v1-only tile)
    if (ver == 1 && v2_first && found) continue;
    for (int tk : tks)
    for (int tw = 1; tw <= 14; ++tw)
    for (int kg : kgs)
    for (int pw = 1; pw * kg <= 16; ++pw)
    for (int tn = 1; tn <= tn_max; tn = (tn < 4 ? tn + 1 : tn * 2))
    for (int bc : bcs)
    for (int fl = 0; fl < 2; ++fl) {
        SimtTile t;
        t.tk = tk; t.tw = tw; t.kg = kg; t.pw = pw; t.tn = tn; t.bc = bc; t.ver = ver;
        if (fl) {
            // flat row mode (whole images, every lane an output row): once
            // per register tile, where the row-mode TMA layout applies
            if (ver != 2 || tn != 1 || tw != pb.W || !simt_v2_tw_ok(pb, tw)) continue;
            t.flat = 1;
            t.th = pb.H;
            t.tn = simt_flat_images(pb, t);
            if (!simt2_layout(pb, t).tma) continue;
        }
        // 2-channel chunks and CTAs under 4 warps: forced only (flat r02c:
        // kg 2 / bc 2 1181 us vs kg 4 / bc 4 1163 on the batched layer, which
        // the model, blind to the per-chunk waits, ranked the other way)
        // (6-channel chunks: flat tiles only, r02e)
        if ((bc == 2 || bc == 12 || (bc == 6 && !t.flat)) && !(forced && (forced_mask & 64))) continue;
        if (t.flat && t.kg * t.pw < 4 && !tile_forced) continue;
        if (forced && (forced_mask & 1024)) t.rem = forced->rem;
        if (forced) {
            if ((forced_mask & 512) && t.flat != forced->flat) continue;
            if ((forced_mask & 1) && t.tk != forced->tk) continue;
            if ((forced_mask & 2) && t.tw != forced->tw) continue;
            if ((forced_mask & 4) && t.kg != forced->kg) continue;
            if ((forced_mask & 8) && t.pw != forced->pw) continue;
            if ((forced_mask & 16) && t.tn != forced->tn) continue;
            if ((forced_mask & 64) && t.bc != forced->bc) continue;
        }
        if (!simt_tile_supported(t)) continue;
        if (ver == 2 && !simt_v2_tw_ok(pb, tw)) continue;
        if (!t.flat) {
        // rows per tile: as many as the pixel slots allow
        const long slots = 32L * pw;                                   // lanes per k-group
        const long per_row = ver == 2 ? (pb.W + tw - 1) / tw : pb.W;   // slots one output row needs
        const long cap = ver == 2 ? slots : slots * tw;
        int th = (int)std::min<long>(pb.H, cap / ((long)tn * per_row));
        if (forced && (forced_mask & 32)) th = forced->th;
        if (th < 1) continue;
        if ((long)tn * th * per_row > cap) continue;
        // slot utilisation >= 50% unless the tile already covers all pixels
        const bool whole = th >= pb.H && tn >= pb.N;
        if (2L * tn * th * per_row < cap && !whole && !(forced && (forced_mask & 32))) continue;
        t.th = th;
        } else if (forced && (forced_mask & 32) && forced->th != pb.H) {
            continue;
        }
        if (simt_smem_bytes(pb, t) > dev.smem_optin) continue;
        if (t.kg > 1 && t.kg * t.tk >= 2 * pb.K && !tile_forced) continue;  // mostly-empty k tile
        // split-C while the grid is small (each CTA would otherwise walk the
        // whole C reduction alone): S partial outputs, summed in split order
        const long ctas = simt_ctas(pb, t, pb.N);
        const int nchunks = (pb.C + bc - 1) / bc;
        // forced tiles: the forced split count (tile key splits), else none
        static const int kSimtSplits[] = {1, 2, 4, 8, 16};
        const int forced_sp[] = {forced ? ((forced_mask & 256) ? forced->splits : 1) : 1};
        const int* cand = forced ? forced_sp : kSimtSplits;
        const int ncand = forced ? 1 : 5;
        for (int ci = 0; ci < ncand; ++ci) {
            const int sp = cand[ci];
            t.splits = sp;
            // (r02e: also a 2-way split of a larger flat grid when it brings the remainder launch --
            // finer CTAs whose last round then runs beside the main grid; batched shards N = 32 / 64:
            // 181 / 319 us vs 202 / 333 for the unsplit picks, profiles/r02e/remsplit/)
            const bool flat_rem2 = t.flat && sp == 2 && ctas * sp <= 8L * dev.sms && simt_rem_tiles(pb, t, dev.sms) > 0;
            if (!forced && sp > 1 && ((ctas * sp > 2L * dev.sms && !flat_rem2) || sp > nchunks)) continue;
            ModelResult r = model_simt(pb, dev, t);
            // near-ties (e.g. tiles at the chunk-latency floor): the tile that
            // issues less (r01b Y23: TK 8 vs 4 both modeled 656 us, measured
            // 1129 vs 1316 us)
            const bool tie = found && fabs(r.model_us - best_r.model_us) <= 0.005 * best_r.model_us;
            // and on equal issue as well, the deeper channel chunk (fewer
            // ring waits / barriers: r02 batched layer bc 8 vs 4, 1303 vs
            // 1348 us; charging every chunk instead -- CONV_SIMT_CHUNK_SYNC --
            // lost 2.6 % on the Table-1 total, profiles/r02/t1_simt_sync*.jsonl)
            const bool issue_tie = tie && fabs(r.issue_cyc - best_r.issue_cyc) <= 0.001 * best_r.issue_cyc;
            // v2 near-ties within 1 % of issue: the finer tile (more resident
            // CTA slots) -- its last CTAs and conv_run_host's chunks balance
            // better (r02b batched: kg 4 vs kg 8 equal on the device, 1.79 vs
            // 1.91 ms end to end, profiles/r02b/e2e_kg8.txt)
            const bool fine_tie = tie && t.ver == 2 && best.ver == 2 && r.ctas != best_r.ctas &&
                                  fabs(r.issue_cyc - best_r.issue_cyc) <= 0.01 * best_r.issue_cyc;
            if (!found || (fine_tie ? r.ctas > best_r.ctas
                           : issue_tie ? t.bc > best.bc
                                       : tie ? r.issue_cyc < best_r.issue_cyc : r.model_us < best_r.model_us)) {
                best = t; best_r = r; found = true;
            }
        }
    }
    }
    if (!found) why = "no SIMT tile fits shared memory for this request";
    return found;
}

}  // namespace conv

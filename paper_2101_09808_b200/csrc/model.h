// model.h -- selector internals (not part of the ABI).
#pragma once
#include <string>

#include "internal.h"

namespace conv {

struct ModelResult {
    long tiles = 0;          // CTA tiles
    long ctas = 0;           // CTAs resident in the first wave
    double wave_eff = 1.0;   // tiles / (waves * slots)
    double t_comp_us = 0;    // issued FLOPs / path peak
    double dv_l2_smem = 0;   // bytes L2 -> SMEM (Sec. 3.2 model, CTA tile)
    double t_l2_us = 0;
    double dv_hbm = 0;       // bytes HBM (compulsory + layout transforms)
    double t_hbm_us = 0;
    double model_us = 0;     // modeled conv_run time
    size_t smem = 0;         // dynamic shared memory per CTA
    double issue_cyc = 0;    // SIMT: per-SM issue cycles before the chunk-latency floor (tie-break)
};

// Tensor-path tile keys forced through conv_plan_set_tile (0 / -1: free).
struct TcForce {
    int bn = 0, stages = 0, cg = 0, kbs = 0, splits = 0;
    int fuse = -1, pre_c = -1;
    int expand = -1;        // tiny-C tap expansion: -1 auto (expand_useful), 0 off, 1 on
    int split = 0;          // FP32_TC piece pairs: 0 default (6), 6 or 9
    int bn_max = 0;         // largest BN considered (0: any)
    int halo = -1;          // halo kernel: -1 auto, 0 off, 1 forced
};

ModelResult model_tc(const Problem& pb, const Device& dev, bool bf16, const TcTile& t);
bool select_tc(const Problem& pb, const Device& dev, bool bf16, TcTile& best, ModelResult& r, const TcForce& f,
               std::string& why);
ModelResult model_simt(const Problem& pb, const Device& dev, const SimtTile& t);
// forced_mask bits: 1 tk, 2 tw, 4 kg, 8 pw, 16 tn, 32 th, 64 bc, 128 ver, 256 splits, 512 flat, 1024 rem
bool select_simt(const Problem& pb, const Device& dev, SimtTile& best, ModelResult& r,
                 const SimtTile* forced, unsigned forced_mask, std::string& why);

}  // namespace conv

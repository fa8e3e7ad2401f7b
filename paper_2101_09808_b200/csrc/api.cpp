// api.cpp -- the C ABI (include/conv.h): plan objects, argument validation,
// path/tile selection, describe JSON, and run dispatch.  No computation of
// Eq. 1 happens on the host; every step of conv_run is a kernel of this
// library, and there is no CPU fallback.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "../../include/conv.h"
#include "internal.h"
#include "model.h"

namespace conv {
PFN_encodeTiled g_encode_tiled = nullptr;
PFN_encodeIm2col g_encode_im2col = nullptr;

bool driver_init(std::string& err) {
    static std::once_flag once;
    static std::string init_err;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            init_err = "cannot resolve cuTensorMapEncodeTiled";
            return;
        }
        g_encode_tiled = reinterpret_cast<PFN_encodeTiled>(fn);
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            init_err = "cannot resolve cuTensorMapEncodeIm2col";
            return;
        }
        g_encode_im2col = reinterpret_cast<PFN_encodeIm2col>(fn);
    });
    err = init_err;
    return init_err.empty();
}
}  // namespace conv

using namespace conv;

struct conv_plan {
    Problem pb;
    bool expand = false;    // tensor paths: run expanded_problem(pb) after the tap expansion
    Problem pe{};
    int split = 0;          // FP32_TC: piece pairs (6 or 9); the kernel runs split_problem(pb, split)
    Problem ps{};
    Device dev;
    conv_path requested = CONV_PATH_AUTO;
    conv_path path = CONV_PATH_AUTO;
    TcTile tc;
    TcLayout tcl;
    SimtTile simt;
    ModelResult model;
    // forced tile (conv_plan_set_tile)
    TcForce force_tc;
    SimtTile force_simt;
    unsigned force_simt_mask = 0;
    // conv_run_host pipeline (created on first use, guarded by host_mu)
    std::mutex host_mu;
    cudaStream_t h2d = nullptr, comp = nullptr, comp2 = nullptr, d2h = nullptr;   // comp2: FP32 SIMT chunks alternate
    static constexpr int kMaxChunks = 32;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_h2d[kMaxChunks] = {}, ev_comp[kMaxChunks] = {};
    int host_nch = 0;                           // image chunks of the pipeline (0: not planned yet)
    SimtTile simt_host;                         // FP32 SIMT: the tile the pipeline's chunks run with (compute_host_chunks)
    int host_bounds[kMaxChunks + 1] = {};       // chunk j = images [host_bounds[j], host_bounds[j+1])
    ~conv_plan() {
        for (cudaStream_t s : {h2d, comp, comp2, d2h}) if (s) cudaStreamDestroy(s);
        for (cudaEvent_t e : {ev_start, ev_end}) if (e) cudaEventDestroy(e);
        for (int i = 0; i < kMaxChunks; ++i) {
            if (ev_h2d[i]) cudaEventDestroy(ev_h2d[i]);
            if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
        }
    }
};

static thread_local std::string g_err;
static thread_local conv_status g_status = CONV_OK;

static conv_status fail(conv_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    g_status = s;
    return s;
}

extern "C" const char* conv_last_error(void) { return g_err.c_str(); }
extern "C" conv_status conv_last_status(void) { return g_status; }
#ifndef CONV_ENABLE_TRACE
#define CONV_ENABLE_TRACE 0
#endif
extern "C" const char* conv_version(void) { return CONV_ENABLE_TRACE ? "0.1.0 sm_100a +trace" : "0.1.0 sm_100a"; }

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

static size_t ws_bytes(const conv_plan* p) {
    if (p->path == CONV_PATH_FP32_SIMT) return align256(simt_ws_bytes(p->pb, p->simt));
    if (p->tc.halo) return align256(halo_ws_bytes(p->pb, p->path == CONV_PATH_BF16));   // the B image only
    // aux region: the fused transform's flags, or split-K's counters + partials
    const Problem& kp = p->split ? p->ps : (p->expand ? p->pe : p->pb);   // the problem the tensor kernel runs
    const size_t aux = p->tc.fuse ? p->tcl.flag_bytes : tc_split_bytes(kp, p->tcl, p->tc);
    return align256(p->tcl.in_ws_bytes) + align256(p->tcl.ker_ws_bytes) + align256(aux);
}

// Tensor-path selection on the problem the kernel will run: tiny-C layers
// (expand_useful, or forced with the tile key expand) run their 1x1
// tap-expanded equivalent, without the fused transform or split-K.
static bool select_tensor(conv_plan* p, bool bf16, TcTile& tt, ModelResult& rt, bool& expand, Problem& pe,
                          std::string& why) {
    const Problem& pb = p->pb;
    // automatic only when the fused transform / split-K are not forced
    expand = p->force_tc.expand >= 0 ? p->force_tc.expand == 1
                                     : expand_useful(pb, bf16) && p->force_tc.fuse != 1 && p->force_tc.splits <= 1 &&
                                           p->force_tc.halo != 1;
    if (expand && (p->force_tc.fuse == 1 || p->force_tc.splits > 1)) {
        why = "the tap expansion runs without the fused transform and split-K";
        return false;
    }
    if (!expand) return select_tc(pb, p->dev, bf16, tt, rt, p->force_tc, why);
    pe = expanded_problem(pb);
    TcForce f = p->force_tc;
    f.fuse = 0;
    f.splits = 1;
    f.halo = 0;                                   // the halo kernel reads the real NCHW input
    if (!select_tc(pe, p->dev, bf16, tt, rt, f, why)) return false;
    // the expansion reads In (fp32) and Ker and writes the expanded workspace
    // instead of the plain repack the model charged for pe
    return true;
}

// FP32_TC layout: the bf16 layout of the split problem; when each piece
// block is whole k-blocks the NHWC workspace holds the 3 pieces once (3*Cq
// channels, half of the 6-pair layout) and the kernel maps pair blocks to
// pieces (tc_run)
static TcLayout split_layout(const Problem& real, const Problem& ps) {
    TcLayout L = tc_layout(ps, true);
    // default since r02c (env CONV_SPLIT_COMPACT=0: the 6-pair layout): on
    // the batched layer the compact layout's transform is 16-18 us shorter
    // (35 vs 52-55 us) and its main kernel ~5 % longer (262-264 vs 249-263
    // us); r02 measured that a wash (186-200 vs 194-200 TFLOP/s), r02c
    // 200.8-202.5 vs 190.0-197.9 TFLOP/s over three alternations on one box
    // (profiles/r02c/ab/)
    static const bool compact = !(getenv("CONV_SPLIT_COMPACT") && atoi(getenv("CONV_SPLIT_COMPACT")) == 0);
    if (compact && split_compact_ok(real, L.bkc)) {
        L.a_chan = 3 * split_cq(real.C);
        L.in_ws_bytes = (size_t)real.N * real.Hin() * real.Win() * L.a_chan * L.elem;
    }
    return L;
}

// FP32_TC selection: the bf16 kernel's tiles on split_problem(pb, npairs)
// (no fused transform, no tap expansion).  The model charged the layout
// transform the fp32 read of npairs*Cq input channels; the split launch reads
// the C real ones once.
static bool select_split(conv_plan* p, TcTile& tt, ModelResult& rt, Problem& ps, int& np, std::string& why) {
    np = p->force_tc.split ? p->force_tc.split : 6;
    ps = split_problem(p->pb, np);
    TcForce f = p->force_tc;
    if (f.fuse == 1) { why = "FP32_TC plans run without the fused transform"; return false; }
    f.fuse = 0;
    f.expand = 0;
    f.halo = 0;                                   // the halo kernel reads the real NCHW input
    if (!select_tc(ps, p->dev, true, tt, rt, f, why)) return false;
    const double over = 4.0 * ((double)ps.in_elems() - (double)p->pb.in_elems()) +
                        4.0 * ((double)ps.ker_elems() - (double)p->pb.ker_elems());
    rt.dv_hbm -= over;
    rt.t_hbm_us = rt.dv_hbm / p->dev.bw_hbm * 1e6;
    rt.model_us -= over / (0.8 * p->dev.bw_hbm) * 1e6;
    return true;
}

// Re-run the selector for the requested path (Alg. 1:
// every candidate evaluated, minimum modeled cost wins).
static conv_status select(conv_plan* p) {
    std::string why;
    p->host_nch = 0;                              // the host pipeline is re-planned for the new tile
    const Problem& pb = p->pb;
    TcTile tt;
    ModelResult rt;
    SimtTile st;
    ModelResult rs;
    const SimtTile* fs = p->force_simt_mask ? &p->force_simt : nullptr;
    p->split = 0;
    switch (p->requested) {
        case CONV_PATH_FP32_SIMT:
            if (!select_simt(pb, p->dev, st, rs, fs, p->force_simt_mask, why)) return fail(CONV_ERR_INFEASIBLE, "%s", why.c_str());
            p->simt = st; p->model = rs; p->path = CONV_PATH_FP32_SIMT;
            break;
        case CONV_PATH_FP32_TC: {
            Problem ps{};
            int np = 0;
            if (!select_split(p, tt, rt, ps, np, why)) return fail(CONV_ERR_INFEASIBLE, "%s", why.c_str());
            p->tc = tt; p->model = rt; p->path = CONV_PATH_FP32_TC; p->expand = false; p->split = np; p->ps = ps;
            p->tcl = split_layout(pb, ps);
            break;
        }
        case CONV_PATH_TF32:
        case CONV_PATH_BF16: {
            const bool bf16 = p->requested == CONV_PATH_BF16;
            bool ex = false;
            Problem pe{};
            if (!select_tensor(p, bf16, tt, rt, ex, pe, why)) return fail(CONV_ERR_INFEASIBLE, "%s", why.c_str());
            p->tc = tt; p->model = rt; p->path = p->requested; p->expand = ex; p->pe = pe;
            p->tcl = tc_layout(ex ? pe : pb, bf16);
            break;
        }
        case CONV_PATH_AUTO:
        default: {
            // AUTO returns results at the paper's precision (fp32, PAPER.md:369;
            // DESIGN.md reading R6): the faster of the FP32 SIMT path and the
            // FP32-accurate tensor path by modeled time.  TF32 / BF16 inputs
            // (relL2 ~3e-4 / ~2e-3) only when requested.
            const bool ok_s = select_simt(pb, p->dev, st, rs, fs, p->force_simt_mask, why);
            Problem ps{};
            int np = 0;
            std::string why_t;
            const bool ok_t = select_split(p, tt, rt, ps, np, why_t);
            if (!ok_s && !ok_t) return fail(CONV_ERR_INFEASIBLE, "%s; %s", why.c_str(), why_t.c_str());
            // The two models are calibrated separately; against the measured
            // Table-1 steps the FP32_TC model reads ~1.2x optimistic relative
            // to the SIMT one (r02, profiles/r02/t1_*_sk.jsonl: AUTO total
            // 1742 us with factor 1.0, 1651 with 1.2, 1688 with 1.4; the
            // per-layer best of the two 1613)
            constexpr double kTcVsSimt = 1.2;
            if (ok_t && (!ok_s || rt.model_us * kTcVsSimt < rs.model_us)) {
                p->tc = tt; p->model = rt; p->path = CONV_PATH_FP32_TC; p->expand = false; p->split = np; p->ps = ps;
                p->tcl = split_layout(pb, ps);
            } else {
                p->simt = st; p->model = rs; p->path = CONV_PATH_FP32_SIMT;
            }
        }
    }
    return CONV_OK;
}

// Plan creation shared by the public constructors: validates the problem,
// binds the current device (or the described offline one) and runs the
// selector.
static conv_plan* create_impl(const Problem& pb, const Device* offline) {
    const int64_t lim = (int64_t)1 << 31;
    if (pb.in_elems() >= lim || pb.ker_elems() >= lim || pb.out_elems() >= lim || pb.Hin() >= lim || pb.Win() >= lim) {
        fail(CONV_ERR_INVALID_ARGUMENT, "tensor with >= 2^31 elements is not supported");
        return nullptr;
    }
    conv_plan* p = new conv_plan();
    p->pb = pb;
    if (offline) {
        p->dev = *offline;
        p->dev.ordinal = -1;                 // not bound to a device: cannot run
    } else {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) {
            cudaGetLastError();
            delete p;
            fail(CONV_ERR_UNSUPPORTED_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
            return nullptr;
        }
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
            delete p;
            fail(CONV_ERR_UNSUPPORTED_DEVICE, "cudaGetDeviceProperties failed");
            return nullptr;
        }
        if (prop.major != 10 || prop.minor != 0) {
            delete p;
            fail(CONV_ERR_UNSUPPORTED_DEVICE, "device %s is sm_%d%d; this library is built for sm_100a only",
                 prop.name, prop.major, prop.minor);
            return nullptr;
        }
        std::string err;
        if (!driver_init(err)) {
            delete p;
            fail(CONV_ERR_UNSUPPORTED_DEVICE, "%s", err.c_str());
            return nullptr;
        }
        p->dev.ordinal = dev;
        p->dev.sms = prop.multiProcessorCount;
        p->dev.cc_major = prop.major;
        p->dev.cc_minor = prop.minor;
        p->dev.smem_optin = prop.sharedMemPerBlockOptin;
        p->dev.l2_bytes = prop.l2CacheSize;
    }
    if (select(p) != CONV_OK) {
        delete p;
        return nullptr;
    }
    return p;
}

static bool strided_problem(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D, int ph, int pw,
                            Problem& pb) {
    if (N < 1 || K < 1 || C < 1 || R < 1 || S < 1 || U < 1 || D < 1 || Hin < 1 || Win < 1) {
        fail(CONV_ERR_INVALID_ARGUMENT, "extent must be >= 1 (N=%d K=%d C=%d Hin=%d Win=%d R=%d S=%d U=%d D=%d)", N, K,
             C, Hin, Win, R, S, U, D);
        return false;
    }
    if (ph < 0 || pw < 0) {
        fail(CONV_ERR_INVALID_ARGUMENT, "padding must be >= 0 (ph=%d pw=%d)", ph, pw);
        return false;
    }
    const int64_t Re = (int64_t)D * (R - 1) + 1, Se = (int64_t)D * (S - 1) + 1;   // dilated kernel extents
    const int64_t Hp = (int64_t)Hin + 2 * (int64_t)ph, Wp = (int64_t)Win + 2 * (int64_t)pw;   // padded input
    if (Hp < Re || Wp < Se) {
        fail(CONV_ERR_INVALID_ARGUMENT, "input %lldx%lld (padded) smaller than the kernel %lldx%lld (dilated extents)",
             (long long)Hp, (long long)Wp, (long long)Re, (long long)Se);
        return false;
    }
    if ((Hp - Re) / U + 1 >= INT32_MAX || (Wp - Se) / U + 1 >= INT32_MAX) {
        fail(CONV_ERR_INVALID_ARGUMENT, "output extent too large");
        return false;
    }
    pb = Problem{N, K, C, (int)((Hp - Re) / U + 1), (int)((Wp - Se) / U + 1), R, S};
    pb.U = U;
    pb.D = D;
    pb.ph = ph;
    pb.pw = pw;
    pb.hin = Hin;
    pb.win = Win;
    return true;
}

extern "C" conv_plan* conv_plan_create(int N, int K, int C, int H, int W, int R, int S) {
    if (N < 1 || K < 1 || C < 1 || H < 1 || W < 1 || R < 1 || S < 1) {
        fail(CONV_ERR_INVALID_ARGUMENT, "extent must be >= 1 (N=%d K=%d C=%d H=%d W=%d R=%d S=%d)", N, K, C, H, W, R, S);
        return nullptr;
    }
    return create_impl(Problem{N, K, C, H, W, R, S}, nullptr);
}

extern "C" conv_plan* conv_plan_create_strided(int N, int K, int C, int Hin, int Win, int R, int S, int U) {
    return conv_plan_create_dilated(N, K, C, Hin, Win, R, S, U, 1);
}

extern "C" conv_plan* conv_plan_create_dilated(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D) {
    return conv_plan_create_padded(N, K, C, Hin, Win, R, S, U, D, 0, 0);
}

extern "C" conv_plan* conv_plan_create_padded(int N, int K, int C, int Hin, int Win, int R, int S, int U, int D,
                                              int ph, int pw) {
    Problem pb;
    if (!strided_problem(N, K, C, Hin, Win, R, S, U, D, ph, pw, pb)) return nullptr;
    return create_impl(pb, nullptr);
}

static bool offline_device(int sms, size_t smem_optin, size_t l2_bytes, Device& d) {
    if (sms < 2 || smem_optin < 16384 || l2_bytes == 0) {
        fail(CONV_ERR_INVALID_ARGUMENT, "device description out of range");
        return false;
    }
    d.sms = sms;
    d.smem_optin = smem_optin;
    d.l2_bytes = l2_bytes;
    return true;
}

extern "C" conv_plan* conv_plan_create_offline(int N, int K, int C, int H, int W, int R, int S, int sms,
                                                size_t smem_optin, size_t l2_bytes) {
    if (N < 1 || K < 1 || C < 1 || H < 1 || W < 1 || R < 1 || S < 1) {
        fail(CONV_ERR_INVALID_ARGUMENT, "extent must be >= 1 (N=%d K=%d C=%d H=%d W=%d R=%d S=%d)", N, K, C, H, W, R, S);
        return nullptr;
    }
    Device d;
    if (!offline_device(sms, smem_optin, l2_bytes, d)) return nullptr;
    return create_impl(Problem{N, K, C, H, W, R, S}, &d);
}

extern "C" conv_plan* conv_plan_create_strided_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                        int sms, size_t smem_optin, size_t l2_bytes) {
    return conv_plan_create_dilated_offline(N, K, C, Hin, Win, R, S, U, 1, sms, smem_optin, l2_bytes);
}

extern "C" conv_plan* conv_plan_create_dilated_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                        int D, int sms, size_t smem_optin, size_t l2_bytes) {
    return conv_plan_create_padded_offline(N, K, C, Hin, Win, R, S, U, D, 0, 0, sms, smem_optin, l2_bytes);
}

extern "C" conv_plan* conv_plan_create_padded_offline(int N, int K, int C, int Hin, int Win, int R, int S, int U,
                                                       int D, int ph, int pw, int sms, size_t smem_optin,
                                                       size_t l2_bytes) {
    Problem pb;
    if (!strided_problem(N, K, C, Hin, Win, R, S, U, D, ph, pw, pb)) return nullptr;
    Device d;
    if (!offline_device(sms, smem_optin, l2_bytes, d)) return nullptr;
    return create_impl(pb, &d);
}

extern "C" conv_status conv_plan_set_path(conv_plan* p, conv_path path) {
    if (!p) return fail(CONV_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (path < CONV_PATH_AUTO || path > CONV_PATH_FP32_TC) return fail(CONV_ERR_INVALID_ARGUMENT, "unknown path %d", (int)path);
    const conv_path old = p->requested;
    p->requested = path;
    conv_status s = select(p);
    if (s != CONV_OK) {
        p->requested = old;
        select(p);
    }
    return s;
}

extern "C" conv_status conv_plan_set_tile(conv_plan* p, const char* spec) {
    if (!p) return fail(CONV_ERR_INVALID_ARGUMENT, "plan is NULL");
    TcForce ft;
    SimtTile fs;
    unsigned mask = 0;
    if (spec && *spec) {
        std::string s(spec);
        size_t pos = 0;
        while (pos < s.size()) {
            size_t comma = s.find(',', pos);
            if (comma == std::string::npos) comma = s.size();
            std::string kv = s.substr(pos, comma - pos);
            pos = comma + 1;
            if (kv.empty()) continue;
            size_t eq = kv.find('=');
            if (eq == std::string::npos) return fail(CONV_ERR_INVALID_ARGUMENT, "malformed tile spec item '%s'", kv.c_str());
            std::string key = kv.substr(0, eq);
            char* end = nullptr;
            long v = strtol(kv.c_str() + eq + 1, &end, 10);
            const long vmin = (key == "fuse" || key == "pre_c" || key == "expand" || key == "halo" || key == "flat" || key == "rem") ? 0 : 1;
            if (!end || *end || v < vmin || v > 4096) return fail(CONV_ERR_INVALID_ARGUMENT, "bad value in '%s'", kv.c_str());
            if (key == "bn") ft.bn = (int)v;
            else if (key == "stages") ft.stages = (int)v;
            else if (key == "cg") ft.cg = (int)v;
            else if (key == "kbs") ft.kbs = (int)v;
            else if (key == "splits") { ft.splits = (int)v; fs.splits = (int)v; mask |= 256; }
            else if (key == "fuse") ft.fuse = v ? 1 : 0;
            else if (key == "pre_c") ft.pre_c = (int)v;
            else if (key == "expand") ft.expand = v ? 1 : 0;
            else if (key == "split") ft.split = (int)v;
            else if (key == "halo") ft.halo = v ? 1 : 0;
            else if (key == "tk") { fs.tk = (int)v; mask |= 1; }
            else if (key == "tw") { fs.tw = (int)v; mask |= 2; }
            else if (key == "kg") { fs.kg = (int)v; mask |= 4; }
            else if (key == "pw") { fs.pw = (int)v; mask |= 8; }
            else if (key == "tn") { fs.tn = (int)v; mask |= 16; }
            else if (key == "th") { fs.th = (int)v; mask |= 32; }
            else if (key == "bc") { fs.bc = (int)v; mask |= 64; }
            else if (key == "ver") { fs.ver = (int)v; mask |= 128; }
            else if (key == "flat") { fs.flat = v ? 1 : 0; mask |= 512; }
            else if (key == "rem") { fs.rem = v ? 1 : 0; mask |= 1024; }
            else return fail(CONV_ERR_INVALID_ARGUMENT, "unknown tile key '%s'", key.c_str());
        }
        if (ft.bn && ft.bn != 32 && ft.bn != 64 && ft.bn != 128 && ft.bn != 192 && ft.bn != 256)
            return fail(CONV_ERR_INFEASIBLE, "bn must be one of 32, 64, 128, 192, 256");
        if (ft.kbs && (ft.kbs > 9 || ft.kbs == 5))
            return fail(CONV_ERR_INFEASIBLE, "kbs must be 1, 2, 3, 4, 6, 7, 8 or 9");
        if (ft.cg && ft.cg != 1 && ft.cg != 2) return fail(CONV_ERR_INFEASIBLE, "cg must be 1 or 2");
        if (ft.split && ft.split != 6 && ft.split != 9) return fail(CONV_ERR_INFEASIBLE, "split must be 6 or 9");
        if (ft.splits > 16) return fail(CONV_ERR_INFEASIBLE, "splits must be <= 16");
        if (ft.splits > 1 && ft.fuse == 1) return fail(CONV_ERR_INFEASIBLE, "split-K needs fuse=0");
    }
    const TcForce oft = p->force_tc;
    const SimtTile ofs = p->force_simt;
    const unsigned omask = p->force_simt_mask;
    p->force_tc = ft;
    p->force_simt = fs; p->force_simt_mask = mask;
    conv_status s = select(p);
    if (s != CONV_OK) {
        p->force_tc = oft;
        p->force_simt = ofs; p->force_simt_mask = omask;
        select(p);
    }
    return s;
}

extern "C" size_t conv_plan_workspace_bytes(const conv_plan* p) { return p ? ws_bytes(p) : 0; }

extern "C" int conv_plan_num_kernels(const conv_plan* p) {
    if (!p) return -1;
    // tensor paths: layout transform (halo plans: the Ker pack) + main; SIMT: pack + main (+ the split-C reduce)
    return p->path == CONV_PATH_FP32_SIMT ? simt_num_kernels(p->simt) : 2;
}

extern "C" conv_path conv_plan_path(const conv_plan* p) { return p ? p->path : CONV_PATH_AUTO; }

extern "C" void conv_plan_destroy(conv_plan* p) { delete p; }

static const char* path_name(conv_path p) {
    switch (p) {
        case CONV_PATH_FP32_SIMT: return "fp32_simt";
        case CONV_PATH_TF32: return "tf32";
        case CONV_PATH_BF16: return "bf16";
        case CONV_PATH_FP32_TC: return "fp32_tc";
        default: return "auto";
    }
}

static int compute_host_chunks(const conv_plan* p, int* out_bounds, double* out_us, SimtTile* host_tile);
extern "C" int conv_plan_describe(const conv_plan* p, char* buf, size_t cap) {
    if (!p) return -1;
    const Problem& pb = p->pb;
    const ModelResult& m = p->model;
    // FP32_TC: the bf16 tensor peak shared by the split's piece pairs
    const double peak = p->path == CONV_PATH_FP32_SIMT ? p->dev.peak_fp32
                        : p->path == CONV_PATH_BF16  ? p->dev.peak_bf16
                        : p->path == CONV_PATH_FP32_TC ? p->dev.peak_bf16 / p->split
                                                       : p->dev.peak_tf32;
    const double comp_bytes = 4.0 * (pb.in_elems() + pb.ker_elems() + pb.out_elems());
    const double roof_us = std::max(pb.flops() / peak, comp_bytes / p->dev.bw_hbm) * 1e6;
    std::string tile;
    char t[256];
    if (p->path == CONV_PATH_FP32_SIMT) {
        // staging: "tma" (one 4-D TMA box + a bulk Ker copy per chunk) or
        // "cp.async" (per-thread copies; v1, and v2 where Win % 4 != 0)
        const bool tma = p->simt.ver == 2 && simt2_layout(pb, p->simt).tma;
        snprintf(t, sizeof t, "{\"ver\":%d,\"tk\":%d,\"tw\":%d,\"kg\":%d,\"pw\":%d,\"tn\":%d,\"th\":%d,\"bc\":%d,\"splits\":%d,\"flat\":%d,\"rem\":%d,\"threads\":%d,\"staging\":\"%s\"}",
                 p->simt.ver, p->simt.tk, p->simt.tw, p->simt.kg, p->simt.pw, p->simt.tn, p->simt.th, p->simt.bc,
                 p->simt.splits, p->simt.flat, tma ? simt_rem_tiles(pb, p->simt, p->dev.sms) : 0,
                 32 * p->simt.kg * p->simt.pw, tma ? "tma" : "cp.async");
    } else {
        snprintf(t, sizeof t, "{\"bm\":%d,\"bn\":%d,\"cg\":%d,\"kbs\":%d,\"stages\":%d,\"splits\":%d,\"expand\":%d,\"split\":%d,\"halo\":%d,\"fuse\":%d,\"tnb\":%d,\"pre_c\":%d,\"bkc\":%d,\"cp\":%d,\"swizzle\":%d}",
                 128 * p->tc.cg, p->tc.bn, p->tc.cg, p->tc.kbs, p->tc.stages, p->tc.splits, p->expand ? 1 : 0, p->split, p->tc.halo, p->tc.fuse, p->tc.fuse ? p->tc.tnb : 0,
                 p->tc.fuse ? std::min(p->tc.pre_c, p->tcl.Cp) : 0,
                 p->tcl.bkc, p->tcl.Cp, p->tcl.sw);
    }
    tile = t;
    // conv_run_host's image chunks (plan_host_chunks) and their modeled time
    int hb[conv_plan::kMaxChunks + 1];
    double host_us = 0;
    SimtTile host_tile;
    const int hn = compute_host_chunks(p, hb, &host_us, &host_tile);
    std::string chunks = "[";
    for (int j = 0; j < hn; ++j) chunks += (j ? "," : "") + std::to_string(hb[j + 1] - hb[j]);
    chunks += "]";
    char out[2560];
    int n = snprintf(out, sizeof out,
        "{\"problem\":{\"N\":%d,\"K\":%d,\"C\":%d,\"H\":%d,\"W\":%d,\"R\":%d,\"S\":%d,\"U\":%d,\"D\":%d,\"ph\":%d,\"pw\":%d,\"Hin\":%lld,\"Win\":%lld},"
        "\"path\":\"%s\",\"tile\":%s,\"workspace_bytes\":%zu,\"kernels\":%d,"
        "\"model\":{\"tiles\":%ld,\"ctas\":%ld,\"wave_eff\":%.4f,\"smem_bytes\":%zu,"
        "\"levels\":{\"l2_smem\":{\"dv_bytes\":%.12g,\"bw\":%.6g,\"us\":%.4f},"
        "\"hbm\":{\"dv_bytes\":%.12g,\"bw\":%.6g,\"us\":%.4f},"
        "\"compute\":{\"flops_issued_us\":%.4f,\"peak\":%.6g}},\"model_us\":%.4f},"
        "\"roofline\":{\"flops\":%.6g,\"compulsory_bytes\":%.6g,\"roofline_us\":%.4f},"
        "\"host_pipeline\":{\"chunks\":%s,\"model_us\":%.4f,\"simt_kg\":%d},"
        "\"device\":{\"ordinal\":%d,\"sms\":%d,\"smem_optin\":%zu,\"l2_bytes\":%zu}}",
        pb.N, pb.K, pb.C, pb.H, pb.W, pb.R, pb.S, pb.U, pb.D, pb.ph, pb.pw, (long long)pb.Hin(), (long long)pb.Win(), path_name(p->path), tile.c_str(), ws_bytes(p),
        conv_plan_num_kernels(p), m.tiles, m.ctas, m.wave_eff, m.smem,
        m.dv_l2_smem, p->dev.bw_l2, m.t_l2_us, m.dv_hbm, p->dev.bw_hbm, m.t_hbm_us, m.t_comp_us, peak,
        m.model_us, pb.flops(), comp_bytes, roof_us, chunks.c_str(), host_us, p->path == CONV_PATH_FP32_SIMT ? host_tile.kg : 0, p->dev.ordinal, p->dev.sms, p->dev.smem_optin,
        p->dev.l2_bytes);
    if (n < 0) return -1;
    if (buf && cap) {
        size_t c = std::min((size_t)n, cap - 1);
        memcpy(buf, out, c);
        buf[c] = 0;
    }
    return n;
}

static conv_status check_ptr(const void* ptr, const char* name, size_t align) {
    if (!ptr) return fail(CONV_ERR_INVALID_ARGUMENT, "%s is NULL", name);
    if (reinterpret_cast<uintptr_t>(ptr) % align) return fail(CONV_ERR_INVALID_ARGUMENT, "%s is not %zu-B aligned", name, align);
    return CONV_OK;
}

// Launch the plan's kernels for images [n0, n0 + sub.N) of the plan's problem
// (sub = the plan's problem with N replaced).  The tensor paths' NHWC
// workspace slice of those images and the shared Ker workspace are addressed
// inside the plan's full workspace, so chunks never overlap.
static conv_status launch_kernels(const conv_plan* p, const Problem& sub, int n0, const float* in, const float* ker,
                                  float* out, void* ws, cudaStream_t st, cudaEvent_t* evp,
                                  const SimtTile* simt_tile = nullptr, bool simt_skip_pack = false) {
    std::string err;
    cudaError_t e;
    if (p->path == CONV_PATH_FP32_SIMT) {
        e = simt_run(sub, simt_tile ? *simt_tile : p->simt, in, ker, out, ws, st, evp, err, p->dev.sms, simt_skip_pack);
    } else {
        uint8_t* wsb = static_cast<uint8_t*>(ws);
        const size_t per_img = p->tcl.in_ws_bytes / (size_t)p->pb.N;
        void* in_ws = wsb + per_img * (size_t)n0;
        void* ker_ws = p->tc.halo ? ws : wsb + align256(p->tcl.in_ws_bytes);   // halo: the B image
        void* flag_ws = (p->tc.fuse || p->tc.splits > 1) ? wsb + align256(p->tcl.in_ws_bytes) + align256(p->tcl.ker_ws_bytes)
                                                         : nullptr;
        if (p->split) {
            e = tc_run(split_problem(sub, p->split), p->tcl, p->tc, true, in, ker, out, in_ws, ker_ws, flag_ws, st,
                       p->dev.sms, evp, err, &sub, p->split);
        } else if (p->expand) {
            const Problem sub_e = expanded_problem(sub);
            e = tc_run(sub_e, p->tcl, p->tc, p->path == CONV_PATH_BF16, in, ker, out, in_ws, ker_ws, flag_ws, st,
                       p->dev.sms, evp, err, &sub);
        } else {
            e = tc_run(sub, p->tcl, p->tc, p->path == CONV_PATH_BF16, in, ker, out, in_ws, ker_ws, flag_ws, st,
                       p->dev.sms, evp, err);
        }
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(CONV_ERR_CUDA, "%s%s%s", err.c_str(), err.empty() ? "" : ": ", cudaGetErrorString(e));
    }
    return CONV_OK;
}

static conv_status run_impl(const conv_plan* p, const float* in, const float* ker, float* out, void* ws,
                            void* stream, void* const* events, int n_events) {
    if (!p) return fail(CONV_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (p->dev.ordinal < 0) return fail(CONV_ERR_UNSUPPORTED_DEVICE, "offline plan: not bound to a device");
    conv_status s;
    if ((s = check_ptr(in, "in", 16)) != CONV_OK) return s;
    if ((s = check_ptr(ker, "ker", 16)) != CONV_OK) return s;
    if ((s = check_ptr(out, "out", 16)) != CONV_OK) return s;
    const size_t need = ws_bytes(p);
    if (need && (s = check_ptr(ws, "workspace", 256)) != CONV_OK) return s;
    const int nk = conv_plan_num_kernels(p);
    if (events && n_events != nk + 1) return fail(CONV_ERR_INVALID_ARGUMENT, "n_events must be %d", nk + 1);
    // Out must not alias the inputs or the workspace.
    const char* o0 = reinterpret_cast<const char*>(out);
    const char* o1 = o0 + 4 * p->pb.out_elems();
    auto overlaps = [&](const void* b, size_t bytes) {
        const char* a0 = static_cast<const char*>(b);
        return a0 < o1 && o0 < a0 + bytes;
    };
    if (overlaps(in, 4 * p->pb.in_elems()) || overlaps(ker, 4 * p->pb.ker_elems()) || (need && overlaps(ws, need)))
        return fail(CONV_ERR_INVALID_ARGUMENT, "out aliases in, ker or workspace");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != p->dev.ordinal)
        return fail(CONV_ERR_INVALID_ARGUMENT, "current device %d is not the plan's device %d", dev, p->dev.ordinal);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaEvent_t ev[4];                     // up to 3 kernels (split-C SIMT plans) + 1
    cudaEvent_t* evp = nullptr;
    if (events) {
        for (int i = 0; i <= nk; ++i) {
            ev[i] = static_cast<cudaEvent_t>(events[i]);
            const cudaError_t q = ev[i] ? cudaEventQuery(ev[i]) : cudaErrorInvalidResourceHandle;
            if (q != cudaSuccess && q != cudaErrorNotReady) {
                cudaGetLastError();
                return fail(CONV_ERR_INVALID_ARGUMENT, "events[%d] is not a valid cudaEvent_t", i);
            }
        }
        evp = ev;
    }
    return launch_kernels(p, p->pb, 0, in, ker, out, ws, st, evp);
}

extern "C" conv_status conv_run(const conv_plan* p, const float* in, const float* ker, float* out, void* ws,
                                void* stream) {
    return run_impl(p, in, ker, out, ws, stream, nullptr, 0);
}

extern "C" conv_status conv_run_events(const conv_plan* p, const float* in, const float* ker, float* out,
                                       void* ws, void* stream, void* const* events, int n_events) {
    if (!events) return fail(CONV_ERR_INVALID_ARGUMENT, "events is NULL");
    return run_impl(p, in, ker, out, ws, stream, events, n_events);
}

extern "C" size_t conv_plan_host_run_bytes(const conv_plan* p) {
    if (!p) return 0;
    return align256(4 * p->pb.in_elems()) + align256(4 * p->pb.ker_elems()) + align256(4 * p->pb.out_elems()) +
           ws_bytes(p);
}

// ---- conv_run_host chunk plan -----------------------------------------
// The pipeline overlaps the upload of chunk j+1, the convolution of chunk j
// and the download of chunk j-1 on three streams.  Its length is
//   t_h2d(first chunk) + the compute chain + t_d2h(last chunk)
// when compute-bound, or all uploads + the last chunk's compute and download
// when transfer-bound; small chunks at the ends shorten both, but chunks
// that leave SM waves partly empty lengthen the compute chain.  The plan is
// chosen like a tile (Alg. 1: every candidate evaluated
// on the model, the minimum wins): equal partitions into c = 1..32 chunks,
// and the same with a small head and tail chunk, each simulated with the
// selector's model time of every chunk's sub-problem (same tile) and the
// host link measured on the box (r02b profiles/r02b/e2e/: pinned
// H2D 55.2 GB/s, D2H 56.9 GB/s alone; both at once 67 + 51 MB in 1.31 ms,
// i.e. the upload at ~0.92 and the download at ~0.70 of its solo rate --
// the rates below, as the two overlap for most of the pipeline).
static const double kH2dBps = 55.2e9 * 0.92, kD2hBps = 56.9e9 * 0.70, kD2hSoloBps = 56.9e9;
// per chunk beyond the model: copy + event + launch issue; the tensor
// paths' chunks also pay their layout launch and main-kernel prologue again
// (measured r02b, profiles/r02b/e2e/e2e_check.txt: bf16 16 vs 6 equal
// chunks +0.25 ms, i.e. ~25 us per extra chunk)
static const double kChunkOverheadUs = 6.0, kTcChunkOverheadUs = 30.0;

// FP32 SIMT chunk time: measured r02b on the batched layer's tile
// (profiles/r02b/e2e/simt_time_vs_batch.txt, N = 6..256 images) the time is
// T(k) = 35 + 85 k us with k = ceil(CTAs / SMs) -- proportional to the CTAs
// each SM runs, whatever their concurrency (FFMA2 keeps the FMA pipe busy
// from one warp per SMSP, so a lone CTA runs ~3x faster than one of three),
// plus a fixed ~35 us (launch, Ker pack, ring fill and drain).  The chunk
// estimate scales the full problem's model by that: a + (model - a) k/k_full.
static const double kSimtChunkFixedUs = 35.0;
static double model_run_us(const conv_plan* p, const SimtTile& st, const ModelResult& sm, const Problem& sub) {
    if (p->path == CONV_PATH_FP32_SIMT) {
        const int64_t sms = std::max(1, p->dev.sms);
        const int64_t k_sub = (simt_ctas(sub, st, sub.N) + sms - 1) / sms;
        const int64_t k_full = std::max<int64_t>(1, (simt_ctas(p->pb, st, p->pb.N) + sms - 1) / sms);
        const double full = std::max(sm.model_us, kSimtChunkFixedUs + 1.0);
        return kSimtChunkFixedUs + (full - kSimtChunkFixedUs) * (double)k_sub / (double)k_full;
    }
    if (p->split) return model_tc(split_problem(sub, p->split), p->dev, true, p->tc).model_us;
    if (p->expand) return model_tc(expanded_problem(sub), p->dev, p->path == CONV_PATH_BF16, p->tc).model_us;
    return model_tc(sub, p->dev, p->path == CONV_PATH_BF16, p->tc).model_us;
}

static double simulate_host_pipeline(const conv_plan* p, const SimtTile& st, const ModelResult& sm, const int* bounds, int nch) {
    const Problem& pb = p->pb;
    const double img_in = 4.0 * pb.C * pb.Hin() * pb.Win(), img_out = 4.0 * pb.K * pb.H * pb.W;
    double th = 4.0 * pb.ker_elems() / kH2dBps * 1e6, tc = 0, td = 0;
    for (int j = 0; j < nch; ++j) {
        const int n = bounds[j + 1] - bounds[j];
        if (n <= 0) continue;
        Problem sub = pb;
        sub.N = n;
        // (the tensor paths' per-chunk cost shows up on the whole pipeline,
        // measured; it is charged to the upload chain, which sets their pace)
        th += n * img_in / kH2dBps * 1e6 + (p->path == CONV_PATH_FP32_SIMT ? kChunkOverheadUs : kTcChunkOverheadUs);
        tc = std::max(tc, th) + model_run_us(p, st, sm, sub);
        // the last download has the link to itself (the uploads are done)
        const double d2h_bps = j == nch - 1 ? kD2hSoloBps : kD2hBps;
        td = std::max(td, tc) + n * img_out / d2h_bps * 1e6;
    }
    return td;
}

static int compute_host_chunks_for(const conv_plan* p, const SimtTile& st, const ModelResult& sm, int* out_bounds, double* out_us) {
    const int N = p->pb.N;
    static const int env_chunks = [] { const char* e = getenv("CONV_HOST_CHUNKS"); return e ? atoi(e) : 0; }();
    auto equal = [&](int c, int* b) {
        for (int j = 0; j <= c; ++j) b[j] = (int)((int64_t)N * j / c);
    };
    if (env_chunks > 0) {                       // experiments: equal chunks
        const int c = std::min({env_chunks, N, (int)conv_plan::kMaxChunks});
        equal(c, out_bounds);
        if (out_us) *out_us = simulate_host_pipeline(p, st, sm, out_bounds, c);
        return c;
    }
    // CONV_HOST_SPLIT=a,b,... (study): explicit chunk sizes summing to N
    static const char* env_split = getenv("CONV_HOST_SPLIT");
    if (env_split) {
        int c = 0, sum = 0;
        out_bounds[0] = 0;
        for (const char* q = env_split; *q && c < conv_plan::kMaxChunks;) {
            const int v = atoi(q);
            if (v <= 0) break;
            sum += v;
            out_bounds[++c] = std::min(sum, N);
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
        if (c > 0 && sum == N) {
            if (out_us) *out_us = simulate_host_pipeline(p, st, sm, out_bounds, c);
            return c;
        }
    }
    int best[conv_plan::kMaxChunks + 1], cand[conv_plan::kMaxChunks + 1];
    int best_n = 1;
    equal(1, best);
    double best_t = simulate_host_pipeline(p, st, sm, best, 1);
    auto consider = [&](int c) {
        const double t = simulate_host_pipeline(p, st, sm, cand, c);
        if (t < 0.995 * best_t) {               // a clear win only: fewer chunks on near-ties
            best_t = t;
            best_n = c;
            std::copy(cand, cand + c + 1, best);
        }
    };
    // wave-aligned partitions: middle chunks of m whole waves of CTAs (a
    // partly empty wave costs nearly a full one), a head of 0 / 1/8 / 1/4 /
    // 1/2 / 1 wave and the remainder as the tail.  FP32 SIMT plans choose
    // among these only: measured r02b on the batched layer
    // (profiles/r02b/e2e/e2e_explicit_splits.txt) one-wave middle chunks with
    // a small head beat every equal partition (6,54,54,54,54,34: 1.80 ms;
    // 8 x 32: 1.92; 6 x 42-43: 2.11), which the per-chunk model -- exact for
    // isolated kernels, not for back-to-back ones -- ranks the other way
    const bool simt = p->path == CONV_PATH_FP32_SIMT;
    {
        int wimg = 0;                           // images that fill the resident CTA slots once
        if (p->path == CONV_PATH_FP32_SIMT && st.flat) {
            // flat tiles: whole slot tiles (32*pw image rows) x k tiles per wave
            const int64_t per_slot_tile = std::max<int64_t>(1, simt_ctas(p->pb, st, 1) /
                                                                   ((p->pb.H + 32 * st.pw - 1) / (32 * st.pw)));
            const int64_t slot_tiles = std::max<int64_t>(1, sm.ctas / per_slot_tile);
            wimg = (int)std::max<int64_t>(1, slot_tiles * 32 * st.pw / p->pb.H);
        } else if (p->path == CONV_PATH_FP32_SIMT) {
            const int64_t per_ntile = simt_ctas(p->pb, st, st.tn);
            wimg = (int)(std::max<int64_t>(1, sm.ctas / std::max<int64_t>(1, per_ntile))) * st.tn;
        } else if (sm.tiles > 0) {
            wimg = (int)std::floor((double)sm.ctas * N / (double)sm.tiles);
        }
        for (int m = 1; wimg >= 1 && m <= 3; ++m) {
            const int mid = m * wimg;
            for (int hq = 0; hq <= 5; ++hq) {   // heads 0, 1/8, 1/4, 1/2, 1 wave
                if (hq == 4 || (simt && hq != 1)) continue;   // SIMT: the measured 1/8-wave head
                const int head = hq == 0 ? 0 : hq == 1 ? std::max(1, wimg / 8) : std::max(1, wimg * (hq - 1) / 4);
                int c = 0, at = 0;
                cand[0] = 0;
                if (head > 0 && head < N) { at = head; cand[++c] = at; }
                while (N - at > mid && c < conv_plan::kMaxChunks - 1) { at += mid; cand[++c] = at; }
                cand[++c] = N;
                if (c >= 2) consider(c);
            }
        }
    }
    const int cmax = simt && best_n > 1 ? 1 : std::min(N, (int)conv_plan::kMaxChunks);
    for (int c = 2; c <= cmax; ++c) {
        for (int taper = 0; taper < 2; ++taper) {
            if (taper) {
                // head and tail of about half an equal chunk, c - 2 equal chunks between
                if (c < 3) continue;
                const int ht = std::max(1, N / (2 * (c - 1)));
                if (N - 2 * ht < c - 2) continue;
                cand[0] = 0;
                cand[1] = ht;
                for (int j = 1; j <= c - 2; ++j) cand[j + 1] = ht + (int)((int64_t)(N - 2 * ht) * j / (c - 2));
                cand[c] = N;
            } else {
                equal(c, cand);
            }
            consider(c);
        }
    }
    std::copy(best, best + best_n + 1, out_bounds);
    if (out_us) *out_us = best_t;
    return best_n;
}

// The FP32 SIMT tile conv_run_host's chunks run with: the plan's tile, or --
// for a flat tile of more than 4 k groups whose kg was not forced -- the
// same tile with half the k groups when the modeled pipeline is shorter
// with it (finer CTA waves give finer one-wave chunks; every unsplit tile
// accumulates each output in the same order, so the results are the same
// bits).  r02d, batched layer: the kg = 8 tile is faster on the device (1091
// vs 1110 us) but its one-wave chunks are 84 images (e2e 2.00 ms) against 61
// for kg = 4 (1.84 ms).
static int compute_host_chunks(const conv_plan* p, int* out_bounds, double* out_us, SimtTile* host_tile) {
    double t0 = 0;
    int n0 = compute_host_chunks_for(p, p->simt, p->model, out_bounds, &t0);
    SimtTile use = p->simt;
    if (p->path == CONV_PATH_FP32_SIMT && p->simt.flat && p->simt.kg > 4 && p->simt.kg % 2 == 0 &&
        !(p->force_simt_mask & 4)) {
        SimtTile h = p->simt;
        h.kg /= 2;
        if (h.bc == 6) h.bc = 4;                // 6-channel chunks would cost the kg = 4 tile a resident CTA (r02e)
        if (simt_tile_supported(h) && simt_smem_bytes(p->pb, h) <= p->dev.smem_optin &&
            simt_ws_bytes(p->pb, h) <= simt_ws_bytes(p->pb, p->simt)) {
            const ModelResult mh = model_simt(p->pb, p->dev, h);
            int b2[conv_plan::kMaxChunks + 1];
            double t1 = 0;
            const int n1 = compute_host_chunks_for(p, h, mh, b2, &t1);
            if (t1 < t0) {
                std::copy(b2, b2 + n1 + 1, out_bounds);
                n0 = n1; t0 = t1; use = h;
            }
        }
    }
    if (out_us) *out_us = t0;
    if (host_tile) *host_tile = use;
    return n0;
}

static void plan_host_chunks(conv_plan* p) { p->host_nch = compute_host_chunks(p, p->host_bounds, nullptr, &p->simt_host); }

extern "C" conv_status conv_run_host(const conv_plan* cp, const float* in_host, const float* ker_host,
                                     float* out_host, void* dbuf, void* stream) {
    if (!cp) return fail(CONV_ERR_INVALID_ARGUMENT, "plan is NULL");
    conv_plan* p = const_cast<conv_plan*>(cp);   // only the pipeline resources are mutated
    if (!in_host || !ker_host || !out_host) return fail(CONV_ERR_INVALID_ARGUMENT, "host pointer is NULL");
    conv_status s;
    if ((s = check_ptr(dbuf, "device_buffer", 256)) != CONV_OK) return s;
    if (p->dev.ordinal < 0) return fail(CONV_ERR_UNSUPPORTED_DEVICE, "offline plan: not bound to a device");
    const Problem& pb = p->pb;
    const size_t bi = 4 * pb.in_elems(), bk = 4 * pb.ker_elems(), bo = 4 * pb.out_elems();
    char* d = static_cast<char*>(dbuf);
    float* din = reinterpret_cast<float*>(d);
    float* dker = reinterpret_cast<float*>(d + align256(bi));
    float* dout = reinterpret_cast<float*>(d + align256(bi) + align256(bk));
    void* dws = d + align256(bi) + align256(bk) + align256(bo);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // Pipeline over image chunks on three internal streams: the upload of
    // chunk j+1, the convolution of chunk j and the download of chunk j-1
    // overlap (PCIe is full duplex); the chunks are planned once per plan on
    // the model (plan_host_chunks).
    std::lock_guard<std::mutex> g(p->host_mu);
    if (p->host_nch == 0) plan_host_chunks(p);
    const int nch = p->host_nch;
    const int* bounds = p->host_bounds;
    cudaError_t e = cudaSuccess;
    auto ok = [&](cudaError_t r) { if (r != cudaSuccess && e == cudaSuccess) e = r; };
    if (!p->h2d) {
        ok(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
        ok(cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking));
        ok(cudaStreamCreateWithFlags(&p->comp2, cudaStreamNonBlocking));
        ok(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
        ok(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
        ok(cudaEventCreateWithFlags(&p->ev_end, cudaEventDisableTiming));
        for (int i = 0; i < conv_plan::kMaxChunks; ++i) {
            ok(cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming));
            ok(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming));
        }
        if (e != cudaSuccess) { cudaGetLastError(); return fail(CONV_ERR_CUDA, "pipeline setup failed: %s", cudaGetErrorString(e)); }
    }
    // everything after the caller's prior work on `stream`
    ok(cudaEventRecord(p->ev_start, st));
    ok(cudaStreamWaitEvent(p->h2d, p->ev_start, 0));
    ok(cudaStreamWaitEvent(p->comp, p->ev_start, 0));
    ok(cudaStreamWaitEvent(p->comp2, p->ev_start, 0));
    ok(cudaStreamWaitEvent(p->d2h, p->ev_start, 0));
    ok(cudaMemcpyAsync(dker, ker_host, bk, cudaMemcpyHostToDevice, p->h2d));
    const int64_t img_in = (int64_t)pb.C * pb.Hin() * pb.Win(), img_out = (int64_t)pb.K * pb.H * pb.W;
    // Study knob CONV_HOST_TWO_COMP=1 (r02e, FP32 SIMT without split-C): the chunks' kernels alternate
    // between two compute streams, so that a chunk's CTAs fill the SMs while the previous chunk's last
    // ones drain.  Ker is packed once, by the first chunk -- the later chunks skip the pack and read the
    // same packed copy, the second stream starts behind the first chunk -- and nothing else in the
    // workspace is shared (split-C partial slabs would be: those plans keep one compute stream); each
    // output is still one CTA's own sequence of FMAs: the same bits (fuzz_run_host.py, 480 runs).
    // Measured on the batched layer (profiles/r02e/e2e/two_comp_ab.txt, three passes): 1.87 vs 1.85 ms
    // with the planned chunks, 1.79 vs 1.82 with a tapered tail, 1.99 vs 2.07 with 30-image chunks --
    // no gain for the plan, so the single compute stream stays the default.
    static const bool two_env = getenv("CONV_HOST_TWO_COMP") != nullptr;
    const bool two_comp = two_env && p->path == CONV_PATH_FP32_SIMT && p->simt_host.splits <= 1 && nch >= 3;
    int n0 = 0, launched = 0;
    for (int j = 0; j < nch && e == cudaSuccess; ++j) {
        const int n1 = bounds[j + 1];
        if (n1 == n0) continue;
        Problem sub = pb;
        sub.N = n1 - n0;
        cudaStream_t cs = (two_comp && (launched & 1)) ? p->comp2 : p->comp;
        ok(cudaMemcpyAsync(din + n0 * img_in, in_host + n0 * img_in, 4 * sub.N * img_in, cudaMemcpyHostToDevice, p->h2d));
        ok(cudaEventRecord(p->ev_h2d[j], p->h2d));
        ok(cudaStreamWaitEvent(cs, p->ev_h2d[j], 0));
        if (e != cudaSuccess) break;
        s = launch_kernels(p, sub, n0, din + n0 * img_in, dker, dout + n0 * img_out, dws, cs, nullptr,
                           p->path == CONV_PATH_FP32_SIMT ? &p->simt_host : nullptr, two_comp && launched > 0);
        if (s != CONV_OK) return s;
        ok(cudaEventRecord(p->ev_comp[j], cs));
        if (two_comp && launched == 0) ok(cudaStreamWaitEvent(p->comp2, p->ev_comp[j], 0));   // packed Ker complete
        ++launched;
        ok(cudaStreamWaitEvent(p->d2h, p->ev_comp[j], 0));
        ok(cudaMemcpyAsync(out_host + n0 * img_out, dout + n0 * img_out, 4 * sub.N * img_out, cudaMemcpyDeviceToHost, p->d2h));
        n0 = n1;
    }
    // the caller's stream continues after the last download (and everything
    // else, which the download depends on)
    ok(cudaEventRecord(p->ev_end, p->d2h));
    ok(cudaStreamWaitEvent(st, p->ev_end, 0));
    if (e != cudaSuccess) { cudaGetLastError(); return fail(CONV_ERR_CUDA, "host pipeline failed: %s", cudaGetErrorString(e)); }
    return CONV_OK;
}

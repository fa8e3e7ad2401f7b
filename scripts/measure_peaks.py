"""Measure this B200's peaks (the paper takes its model's
bandwidths from synthetic benchmarks on the machine, Sec. 7) and
write

  profiles/peaks_measured.json                        (every number + clocks + method)
  paper_2101_09808_b200/csrc/peaks_measured.inc       (the selector's constants)

Probes (libconv_probes.so, include/conv_probes.h), each timed with CUDA events
on the launching stream after warm-up, best of `--reps` bursts and a
back-to-back loop of `--sustain` seconds, NVML clocks sampled during both:

  ffma        FP32 FFMA issue rate, register operands        -> FP32 SIMT "alu" peak
  mma         tcgen05.mma kind::f16 (bf16) / kind::tf32 issue rate, cg 1 and 2
  l2_bulk     L2 -> SMEM, cp.async.bulk, L2-resident 32 MB buffer
  l2_tiled    L2 -> SMEM, 2-D tiled TMA 128x128 B boxes (128-B swizzle)
and the library-level cross-checks of the same kind as MEASURED_PEAKS.json
(the driver's): cuBLAS GEMM 8192^3 in bf16, tf32 (fp32 inputs, TF32 math) and
fp32 (SGEMM), and a torch copy of 1 Gi bf16 elements (HBM).

    python scripts/measure_peaks.py [--reps 10] [--sustain 2.0]
"""
from __future__ import annotations

import argparse
import ctypes
import datetime
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_09808_b200 import build  # noqa: E402
from paper_2101_09808_b200.clocks import ClockSampler  # noqa: E402

OUT_JSON = os.path.join(ROOT, "profiles", "peaks_measured.json")
OUT_INC = os.path.join(ROOT, "paper_2101_09808_b200", "csrc", "peaks_measured.inc")


def load_probes():
    build.build()
    lib = ctypes.CDLL(build.PROBES_LIB)
    vp, i, d, sz, u = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_uint
    for name, res, args in (
        ("probe_ffma", i, [vp, i, i, i, vp]), ("probe_ffma_flops", d, [i, i, i]),
        ("probe_ffma2", i, [vp, i, i, i, vp]),
        ("probe_mma", i, [i, i, i, i, vp, vp]), ("probe_mma_flops", d, [i, i, i, i]),
        ("probe_l2_bulk", i, [vp, sz, i, u, i, vp]), ("probe_l2_tiled", i, [vp, sz, i, i, vp]),
        ("probe_l2_tiled_bytes", d, [i, i]),
    ):
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def timed(launch, reps, sustain_s, dev):
    """(best burst seconds, mean sustained seconds, clocks) of launch()."""
    st = torch.cuda.current_stream(dev)
    for _ in range(3):
        launch(st)
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev.index or 0)
    clk.start()
    burst = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        launch(st)
        b.record(st)
        b.synchronize()
        burst.append(a.elapsed_time(b) * 1e-3)
        time.sleep(0.05)          # bursts: let the power / clock state recover between them
    sus = []
    if sustain_s > 0:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        n = max(1, int(sustain_s / max(min(burst), 1e-6)))
        a.record(st)
        for _ in range(n):
            launch(st)
        b.record(st)
        b.synchronize()
        sus.append(a.elapsed_time(b) * 1e-3 / n)
    clk.stop()
    return min(burst), (float(np.mean(sus)) if sus else None), clk.summary()


def rec(kind, unit, amount, best, sus, clocks, note, scale=1e12):
    r = {"value": round(amount / best / scale, 2), "unit": unit, "burst_s": best,
         "sustained": round(amount / sus / scale, 2) if sus else None, "clocks": clocks, "how": note}
    print(f"{kind:>16}: {r['value']:>9} {unit} burst, {r['sustained']} sustained, sm {clocks.get('sm_mhz')} MHz",
          flush=True)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sustain", type=float, default=2.0)
    ap.add_argument("--no-write", action="store_true")
    ap.add_argument("--only", default=None, help="comma-separated probe keys to run (study; implies --no-write)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    lib = load_probes()
    res = {}
    only = set(args.only.split(",")) if args.only else None

    def want(k):
        return only is None or k in only

    def chk(rc, what):
        if rc != 0:
            raise SystemExit(f"{what} failed ({rc})")

    # ---- FFMA: 4 CTAs x 256 threads per SM (32 warps, 16 chains each)
    out = torch.empty(sms * 4 * 256, device=dev)
    if want("ffma"):
        ffma_probes(lib, res, out, sms, args, dev, chk)
    if want("mma"):
        mma_probes(lib, res, sms, args, dev, chk)
    if want("l2"):
        l2_probes(lib, res, sms, args, dev, chk)
    if want("lib"):
        lib_probes(res, args, dev)
    if only is not None:
        print(json.dumps({k: {"value": v["value"], "unit": v["unit"], "clocks": v["clocks"].get("sm_mhz")}
                          for k, v in res.items()}))
        return
    finish(res, sms, args, dev)


def ffma_probes(lib, res, out, sms, args, dev, chk):
    blocks, threads, iters = sms * 4, 256, 4000
    fl = lib.probe_ffma_flops(blocks, threads, iters)
    b, s, c = timed(lambda st: chk(lib.probe_ffma(out.data_ptr(), blocks, threads, iters, st.cuda_stream), "ffma"),
                    args.reps, args.sustain, dev)
    res["ffma_fp32"] = rec("ffma", "TFLOP/s", fl, b, s, c,
                           f"{blocks}x{threads} threads, 16 register-operand FFMA chains each, 8*{iters} steps")
    sm_clk = c.get("sm_mhz") or 1965.0
    res["ffma_fp32"]["flop_per_clk_per_sm"] = round(fl / b / (sm_clk * 1e6) / sms, 1)

    b, s, c = timed(lambda st: chk(lib.probe_ffma2(out.data_ptr(), blocks, threads, iters, st.cuda_stream), "ffma2"),
                    args.reps, args.sustain, dev)
    res["ffma2_fp32"] = rec("ffma2", "TFLOP/s", fl, b, s, c,
                            f"{blocks}x{threads} threads, 8 register-pair FFMA2 (fma.rn.f32x2) chains each, "
                            f"pair x broadcast scalar, 8*{iters} steps")



def mma_probes(lib, res, sms, args, dev, chk):
    for bf16 in (1, 0):
        for cg in (1, 2):
            iters = 6000 if bf16 else 3000
            grid = (sms // cg) * cg
            fl = lib.probe_mma_flops(bf16, cg, grid, iters)
            b, s, c = timed(lambda st: chk(lib.probe_mma(bf16, cg, grid, iters, None, st.cuda_stream), "mma"),
                            args.reps, args.sustain, dev)
            key = f"mma_{'bf16' if bf16 else 'tf32'}_cg{cg}"
            res[key] = rec(key, "TFLOP/s", fl, b, s, c,
                           f"tcgen05.mma.cta_group::{cg}.kind::{'f16 (bf16)' if bf16 else 'tf32'} M={128 * cg} N=256 "
                           f"K={16 if bf16 else 8}, smem operands, {grid} CTAs, {4 * iters} MMAs each")
            clk = c.get("sm_mhz") or 1965.0
            res[key]["flop_per_clk_per_sm"] = round(fl / b / (clk * 1e6) / grid, 1)



def l2_probes(lib, res, sms, args, dev, chk):
    buf = torch.randint(0, 255, (32 << 20,), dtype=torch.uint8, device=dev)
    buf.sum()                                   # resident in L2
    chunk, iters = 32768, 3000
    by = float(sms * iters * chunk)
    b, s, c = timed(lambda st: chk(lib.probe_l2_bulk(buf.data_ptr(), buf.numel(), sms, chunk, iters,
                                                     st.cuda_stream), "l2_bulk"), args.reps, args.sustain, dev)
    res["l2_smem_bulk"] = rec("l2_bulk", "TB/s", by, b, s, c,
                              f"cp.async.bulk 32 KB x 6 in flight per SM, {sms} CTAs, 32 MB L2-resident source")
    iters = 3000
    by = lib.probe_l2_tiled_bytes(sms, iters)
    b, s, c = timed(lambda st: chk(lib.probe_l2_tiled(buf.data_ptr(), buf.numel(), sms, iters, st.cuda_stream),
                                   "l2_tiled"), args.reps, args.sustain, dev)
    res["l2_smem_tiled"] = rec("l2_tiled", "TB/s", by, b, s, c,
                               f"2-D tiled TMA 128x128 B boxes, 128-B swizzle, 2 boxes x 6 stages in flight, {sms} CTAs")
    del buf



def lib_probes(res, args, dev):
    """library cross-checks (the driver's method for MEASURED_PEAKS.json)"""
    n = 8192
    for name, dt, tf32 in (("cublas_bf16", torch.bfloat16, False), ("cublas_tf32", torch.float32, True),
                           ("cublas_fp32", torch.float32, False)):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        x = torch.randn(n, n, device=dev, dtype=dt)
        y = torch.randn(n, n, device=dev, dtype=dt)
        z = torch.empty(n, n, device=dev, dtype=dt)
        b, s, c = timed(lambda st: torch.matmul(x, y, out=z), args.reps, args.sustain, dev)
        res[name] = rec(name, "TFLOP/s", 2.0 * n ** 3, b, s, c, f"torch.matmul {n}^3 {dt}, allow_tf32={tf32}")
        del x, y, z
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    a2 = torch.empty_like(a)
    b, s, c = timed(lambda st: a2.copy_(a), args.reps, 0, dev)
    res["hbm_copy"] = rec("hbm_copy", "GB/s", 4.0 * (1 << 30), b, s, c, "b.copy_(a), 1 Gi bf16 (read + write bytes)",
                          scale=1e9)
    del a, a2


def finish(res, sms, args, dev):
    doc = {
        "gpu": torch.cuda.get_device_name(dev), "sms": sms, "when": datetime.datetime.now(datetime.timezone.utc).isoformat(),
        "torch": torch.__version__, "probes": res,
        "note": "burst = best of --reps single launches (CUDA events, 50 ms apart); sustained = back-to-back loop "
                f"of ~{args.sustain} s; clocks = NVML samples over both",
    }
    # the constants the selector and bench use
    doc["selected"] = {
        "peak_fp32_tflops": res["ffma_fp32"]["value"],
        "peak_tf32_tflops": res["cublas_tf32"]["value"],
        "peak_tf32_mma_tflops": max(res["mma_tf32_cg1"]["value"], res["mma_tf32_cg2"]["value"]),
        "peak_bf16_mma_tflops": max(res["mma_bf16_cg1"]["value"], res["mma_bf16_cg2"]["value"]),
        "bw_l2_smem_tbs": res["l2_smem_tiled"]["value"],
    }
    print(json.dumps(doc["selected"]))
    if args.no_write:
        return
    os.makedirs(os.path.dirname(OUT_JSON), exist_ok=True)
    with open(OUT_JSON, "w") as f:
        json.dump(doc, f, indent=1)
    write_inc(doc)


def write_inc(doc):
    sel = doc["selected"]
    # HBM and the bf16 peak: the driver's MEASURED_PEAKS.json (the contract's
    # roofline denominators), else this run's own cross-checks
    mp = {}
    mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp_path):
        with open(mp_path) as f:
            mp = json.load(f)
    hbm = mp.get("hbm_gbs", doc["probes"]["hbm_copy"]["value"])
    bf16 = mp.get("bf16_tflops", doc["probes"]["cublas_bf16"]["value"])
    lines = [
        "// peaks_measured.inc -- GENERATED by scripts/measure_peaks.py from",
        "// profiles/peaks_measured.json (probes on a B200 of this pool; DESIGN.md Sec. 6).",
        "// Do not edit by hand: tests/test_abi.py checks it against the JSON.",
        f"// measured {doc['when']} on {doc['gpu']}",
        "#pragma once",
        f"#define CONV_BW_HBM {hbm}e9            // {'MEASURED_PEAKS.json' if 'hbm_gbs' in mp else 'torch copy'} (B/s)",
        f"#define CONV_PEAK_BF16 {bf16}e12       // {'MEASURED_PEAKS.json' if 'bf16_tflops' in mp else 'cuBLAS bf16'} burst",
        f"#define CONV_PEAK_FP32 {sel['peak_fp32_tflops']}e12        // FFMA probe, burst (flop/s)",
        f"#define CONV_PEAK_TF32 {sel['peak_tf32_tflops']}e12       // cuBLAS TF32 GEMM 8192^3, burst",
        f"#define CONV_BW_L2_SMEM {sel['bw_l2_smem_tbs']}e12        // 2-D tiled TMA, L2-resident (B/s)",
        "",
    ]
    with open(OUT_INC, "w") as f:
        f.write("\n".join(lines))


if __name__ == "__main__":
    main()

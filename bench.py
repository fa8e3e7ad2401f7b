#!/usr/bin/env python
"""bench.py -- conv TFLOP/s of Eq. 1 on B200, BASELINE.json's
metric: 2*N*K*H*W*C*R*S / time, plus % of roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--path tf32|bf16|fp32_simt|auto]
                    [--config batched] [--scaling weak|strong] [--gather] [--impl ours|reference]

A "step" is one conv_run over the workload (all of its kernels: the layout
transforms and the main kernel, PAPER.md:371/425/624 count them).  Timing
follows the paper's protocol: each run is timed individually
on the device with CUDA events on the launching stream, with an L2 flush
(a write of a buffer >= 2x L2) before every run, outside the event pair.
The K timed runs are bracketed by a barrier + synchronize on both sides and
the reported time is the max over ranks.

Multi-GPU (torchrun, one process per GPU, NCCL): the batched layer shards by
batch n (only non-reduction dims are parallelised).  Default
"weak": every rank convolves its own batch of 256 images (independent units,
no data-path collective); "strong": the 256 images are split across ranks.
--gather runs NCCL all_gather_into_tensor of the Out slabs after the timed
region and reports its time separately.

--impl reference times the CPU oracle (oracle/, plain C, double) as it stands
on the host cores, on bounded samples of the same workload, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_09808_b200.clocks import ClockSampler  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, Shape, make_inputs  # noqa: E402

METRIC = "conv TFLOP/s (2*N*K*H*W*C*R*S / time)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


def path_peak(path, peaks):
    """Peak for the dominant kernel's arithmetic (TFLOP/s) and its bound."""
    if path == "bf16":
        return peaks["bf16_tflops"], "tensor", "measured cuBLAS bf16 burst (MEASURED_PEAKS.json)"
    if path == "tf32":
        # kind::tf32 issues at half the kind::f16 rate (nominal 1.1 vs 2.25 PF dense)
        return peaks["bf16_tflops"] * 0.5, "tensor", "measured bf16 burst x 0.5 (nominal tf32/bf16 ratio)"
    # FP32 SIMT: 148 SMs x 128 FFMA lanes x 2 flop x max SM clock
    return 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, "alu", \
        "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (derived)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, world):
    base = CONFIGS[args.config]
    if args.scaling == "strong" and world > 1:
        if base.N % world:
            raise SystemExit(f"N={base.N} not divisible by {world}")
        return base, Shape(base.N // world, base.K, base.C, base.H, base.W, base.R, base.S)
    return base, base


def bench_ours(args):
    import torch.distributed as dist

    from paper_2101_09808_b200 import conv

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    full, sh = workload(args, world)

    # inputs: seeded on the CPU; weak scaling gives every rank its own batch
    if args.scaling == "strong" and world > 1:
        inp_all, ker = make_inputs(full, seed=0)
        inp = inp_all[rank * sh.N:(rank + 1) * sh.N].contiguous()
    else:
        inp, ker = make_inputs(sh, seed=rank)
    inp_h, ker_h = inp.pin_memory(), ker.pin_memory()
    d_in, d_ker = inp_h.to(dev), ker_h.to(dev)
    plan = conv.ConvPlan(*sh.as_tuple(), path=args.path, tile=args.tile)
    desc = plan.describe()
    d_out = plan.new_output(dev)
    ws = plan.new_workspace(dev)
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 << 20)
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_rd = torch.ones(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_out = torch.empty((), dtype=torch.float32, device=dev)

    def l2_flush():
        # write a buffer > L2 (evicts every line), then read another one so
        # the dirty lines of the first pass are written back here, outside
        # the timed events: each step starts with a cold, clean L2
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_out)
    stream = torch.cuda.current_stream(dev)
    nk = plan.num_kernels

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up: W steps, then the same step until >= 1 s has passed so that the
    # clocks settle under this load (the clock sampler runs from here on)
    for _ in range(args.warmup):
        l2_flush()
        plan.run(d_in, d_ker, d_out, ws)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < args.soak:
        for _ in range(20):
            l2_flush()
            plan.run(d_in, d_ker, d_out, ws)
        torch.cuda.synchronize(dev)

    # (1) headline: K steps, each conv_run bracketed by its own event pair.
    #     conv_run is replayed from a CUDA graph (its kernels back to back on
    #     the device, the main kernel's programmatic dependent launch kept),
    #     so host launch latency never shows up in the device timing.
    graph = None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                plan.run(d_in, d_ker, d_out, ws)
            cap.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                plan.run(d_in, d_ker, d_out, ws, stream=cap)
            torch.cuda.synchronize(dev)
            graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # pragma: no cover - fall back to stream launches
            print(f"warning: CUDA graph capture failed ({e}); timing stream launches", file=sys.stderr)
            graph = None
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        l2_flush()                                      # L2 flush, outside the event pair
        step_ev[i][0].record(stream)
        if graph is not None:
            graph.replay()
        else:
            plan.run(d_in, d_ker, d_out, ws)
        step_ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    step_ms = np.array([a.elapsed_time(b) for a, b in step_ev])
    ms = float(step_ms.mean())

    # (2) attribution: K more steps with events between the kernels (this
    #     serialises them), giving each kernel's duration on its stream
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)] for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        l2_flush()
        plan.run_events(d_in, d_ker, d_out, ws, evs[i])
    torch.cuda.synchronize(dev)
    barrier()
    clocks.stop()
    per_kernel = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(nk)] for e in evs])  # ms
    main_ms = float(per_kernel[:, -1].mean())
    attributed_ms = float(per_kernel.sum(axis=1).mean())

    # end-to-end through the C ABI with pinned host buffers (H2D + conv + D2H)
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device=dev)
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(max(1, args.warmup)):
        plan.run_host(inp_h, ker_h, out_h, dbuf)
    torch.cuda.synchronize(dev)
    e2e_ms = []
    barrier()
    for _ in range(args.steps):
        l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.run_host(inp_h, ker_h, out_h, dbuf)
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    torch.cuda.synchronize(dev)
    e2e = float(np.mean(e2e_ms))

    gather = None
    if args.gather and world > 1:
        full_out = torch.empty((world,) + tuple(d_out.shape), dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(full_out, d_out)      # warm-up
        torch.cuda.synchronize(dev)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            dist.all_gather_into_tensor(full_out, d_out)
        b.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = a.elapsed_time(b) / args.steps
        gather = {"ms": g_ms, "bytes_recv_per_gpu": (world - 1) * d_out.numel() * 4}

    # max over ranks
    vals = torch.tensor([ms, main_ms, e2e, gather["ms"] if gather else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, main_ms, e2e, g_ms = vals.tolist()
    if gather:
        gather["ms"] = g_ms

    if rank == 0:
        peaks, peak_src = load_peaks()
        peak, bound, peak_note = path_peak(plan.path, peaks)
        flops_rank = sh.flops
        total_flops = flops_rank * world
        value = total_flops / (ms * 1e-3) / 1e12
        achieved = flops_rank / (main_ms * 1e-3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tkey = f"{args.config}:{plan.path}" + (":fuse" if desc["tile"].get("fuse") else "")
                traffic = json.load(f).get(tkey)
        roof_us = max(sh.flops / (peak * 1e12), sh.compulsory_bytes / (peaks["hbm_gbs"] * 1e9)) * 1e6
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "TFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 5),
            # rank 0's K timed steps: the paper's statistic is the mean;
            # median and a normal 95% CI of the mean beside it
            "step_stats": step_stats(step_ms),
            "higher_is_better": True,
            "scaling": "weak" if (args.scaling == "weak" or world == 1) else "strong",
            "vs_baseline": None,
            "dtype": {"bf16": "bf16", "tf32": "tf32", "fp32_simt": "f32"}[plan.path],
            "data": "synthetic (seeded uniform[-1,1), BASELINE.json configs)",
            "config": {
                "workload": f"{args.config}: N={sh.N} K={sh.K} C={sh.C} out {sh.H}x{sh.W} R={sh.R} S={sh.S} "
                            f"(stride 1, no pad, fp32 NCHW/KCRS){' per rank' if world > 1 else ''}",
                "path": plan.path,
                "tile": desc["tile"],
                "l2": "flushed before every timed step, outside the event pair: write of a 2x-L2 buffer, then a read "
                      "of another 2x-L2 buffer (dirty lines written back before the step: cold, clean L2)",
                "clocks_window": "NVML samples every ~1 ms over the >= 1 s warm-up soak and both timed passes",
                "parallelism": f"n-shard x{world}" if world > 1 else "single GPU",
                "kernels_per_step": nk,
                "launch": "cuda_graph replay of conv_run" if graph is not None else "stream launches",
            },
            "roofline": {
                "bound": bound,
                "achieved": round(achieved, 2),
                "peak": round(peak, 1),
                "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4),
                "traffic": traffic,
                "kernel": "conv_igemm_tcgen05" if plan.path != "fp32_simt" else "conv_direct_simt",
                "kernel_ms": round(main_ms, 5),
                "peak_source": f"{peak_note}; {peak_src}",
                "step_roofline_us": round(roof_us, 3),
                "step_frac": round(roof_us / (ms * 1e3), 4),
                "kernel_share_of_step": round(main_ms / attributed_ms, 4),
                "kernel_ms_each": [round(float(x), 5) for x in per_kernel.mean(axis=0)],
                "timing": "kernel durations from a second K-step pass with events between the kernels",
            },
            "e2e": {
                "value": round(total_flops / (e2e * 1e-3) / 1e12, 3),
                "unit": "TFLOP/s",
                "ms_per_step": round(e2e, 4),
                "h2d_bytes_per_step": 4 * (sh.N * sh.C * sh.Hin * sh.Win + sh.K * sh.C * sh.R * sh.S),
                "d2h_bytes_per_step": 4 * sh.N * sh.K * sh.H * sh.W,
                "api": "conv_run_host (C ABI, pinned host buffers)",
            },
            "gpu_launches": nk * args.steps,
            "clocks": clocks.summary(),
        }
        if gather:
            line["gather"] = gather
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(full, args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def oracle_sample_time(sh: Shape, n_img: int, threads: int):
    import oracle
    inp, ker = make_inputs(Shape(n_img, sh.K, sh.C, sh.H, sh.W, sh.R, sh.S), seed=0)
    x, w = inp.numpy(), ker.numpy()
    t0 = time.perf_counter()
    oracle.conv_eq1(x, w, nthreads=threads)
    return time.perf_counter() - t0


def step_stats(step_ms) -> dict:
    x = np.asarray(step_ms, dtype=np.float64)
    mean = float(x.mean())
    half = float(1.96 * x.std(ddof=1) / np.sqrt(len(x))) if len(x) > 1 else 0.0
    return {"mean_ms": round(mean, 5), "median_ms": round(float(np.median(x)), 5),
            "ci95_ms": [round(mean - half, 5), round(mean + half, 5)],
            "min_ms": round(float(x.min()), 5), "max_ms": round(float(x.max()), 5)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(sh: Shape, args, target_s: float = 10.0):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    workload (the first n images of the batch, sized for ~target_s)."""
    import oracle
    threads = oracle.host_threads()
    used = oracle.num_threads(threads)
    t1 = oracle_sample_time(sh, 1, threads)
    n = int(max(1, min(sh.N, target_s / max(t1, 1e-6))))
    t = oracle_sample_time(sh, n, threads) if n > 1 else t1
    flops = 2.0 * n * sh.K * sh.H * sh.W * sh.C * sh.R * sh.S
    return {"value": round(flops / t / 1e12, 6), "unit": "TFLOP/s", "cores": used, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"first {n} of {sh.N} images of the {args.config} layer ({t:.1f} s, double accumulation, "
                      f"OpenMP over (n,k) planes)"}


def bench_reference(args):
    """--impl reference: the oracle on the host cores, same metric."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    sh = CONFIGS[args.config]
    threads = oracle.host_threads()
    used = oracle.num_threads(threads)
    t1 = oracle_sample_time(sh, 1, threads)
    # each step: a bounded sample so that warmup+steps finish in a few minutes
    n = int(max(1, min(sh.N, 8.0 / max(t1, 1e-6))))
    for _ in range(args.warmup):
        oracle_sample_time(sh, 1, threads)
    ts = [oracle_sample_time(sh, n, threads) for _ in range(args.steps)]
    ms = float(np.mean(ts)) * 1e3
    flops = 2.0 * n * sh.K * sh.H * sh.W * sh.C * sh.R * sh.S
    value = flops / (ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1), BASELINE.json configs)",
        "config": {"workload": f"{args.config}: N={sh.N} K={sh.K} C={sh.C} out {sh.H}x{sh.W} R={sh.R} S={sh.S}",
                   "sample_images_per_step": n},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": used, "kind": "oracle",
                         "cpu": cpu_model(), "sample": f"first {n} of {sh.N} images per step"},
        "step_stats": step_stats(np.asarray(ts) * 1e3),
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_table1(args):
    """--sweep table1: every conv2d layer of PAPER.md:439 Table 1 (batch 1,
    stride 1 or 2, Table 1's input extents), one JSON line per layer and
    path, timed like the headline (CUDA-graph replay of conv_run, L2 flushed
    before every step outside the event pair, CUDA events, after warm-up).
    A NEXT-4 study, not the driver's bench line.
    ``--pad same`` runs the layers as the networks do, zero padding R//2
    (NEXT-2)."""
    from paper_2101_09808_b200 import conv
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peaks, peak_src = load_peaks()
    l2 = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20)
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_rd = torch.ones_like(flush)
    flush_out = torch.empty((), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    paths = [args.path] if args.path != "all" else ["bf16", "tf32", "fp32_simt"]
    names = [n for n in TABLE1 if not args.layers or n in args.layers.split(",")]
    for name in names:
        sh = TABLE1[name]
        if args.pad == "same":
            sh = Shape.strided(sh.N, sh.K, sh.C, sh.Hin, sh.Win, sh.R, sh.S, sh.U, 1, sh.R // 2, sh.S // 2)
        inp, ker = make_inputs(sh, seed=0)
        d_in, d_ker = inp.to(dev), ker.to(dev)
        for path in paths:
            plan = conv.ConvPlan(*sh.as_tuple(), path=path, **sh.plan_kwargs())
            if args.tile and path != "fp32_simt":
                plan.set_tile(args.tile)
            out, ws = plan.new_output(dev), plan.new_workspace(dev)
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                for _ in range(max(3, args.warmup)):
                    plan.run(d_in, d_ker, out, ws, stream=cap)
            cap.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                plan.run(d_in, d_ker, out, ws, stream=cap)
            torch.cuda.synchronize(dev)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                torch.sum(flush_rd, dim=0, out=flush_out)
                ev[i][0].record(stream)
                g.replay()
                ev[i][1].record(stream)
            torch.cuda.synchronize(dev)
            ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
            # per-kernel attribution (events between the kernels, same flush)
            nk = plan.num_kernels
            kev = [[torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)] for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                torch.sum(flush_rd, dim=0, out=flush_out)
                plan.run_events(d_in, d_ker, out, ws, kev[i])
            torch.cuda.synchronize(dev)
            kern_us = [round(float(np.mean([e[j].elapsed_time(e[j + 1]) for e in kev])) * 1e3, 2) for j in range(nk)]
            peak, bound, _ = path_peak(plan.path, peaks)
            roof_us = max(sh.flops / (peak * 1e12), 4.0 * (sh.N * sh.C * sh.Hin * sh.Win + sh.K * sh.C * sh.R * sh.S +
                                                           sh.N * sh.K * sh.H * sh.W) / (peaks["hbm_gbs"] * 1e9)) * 1e6
            d = plan.describe()
            print(json.dumps({
                "layer": name, "path": plan.path, "K": sh.K, "C": sh.C, "Hin": sh.Hin, "R": sh.R, "U": sh.U, "pad": sh.ph,
                "out": [sh.H, sh.W], "gflop": round(sh.flops / 1e9, 4), "step_us": round(ms * 1e3, 2),
                "tflops": round(sh.flops / (ms * 1e-3) / 1e12, 3), "roofline_us": round(roof_us, 3),
                "frac": round(roof_us / (ms * 1e3), 4), "kernels_us": kern_us, "tile": d["tile"],
                "peak_source": peak_src}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--path", default="bf16", choices=["auto", "fp32_simt", "tf32", "bf16", "all"])
    ap.add_argument("--config", default="batched", choices=list(CONFIGS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--soak", type=float, default=1.0, help="seconds of extra warm-up steps before timing")
    ap.add_argument("--no-graph", action="store_true", help="time plain stream launches instead of a CUDA graph replay")
    ap.add_argument("--tile", default=None, help="force a tile (conv_plan_set_tile spec, e.g. 'fuse=0,bn=128'); experiments")
    ap.add_argument("--sweep", default=None, choices=["table1"], help="study mode: every Table-1 layer (one JSON line each)")
    ap.add_argument("--layers", default=None, help="--sweep: comma-separated layer names (default all)")
    ap.add_argument("--pad", default="valid", choices=["valid", "same"],
                    help="--sweep: Table 1 as listed (valid, Eq. 1) or with zero padding R//2 (same)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.sweep:
        bench_table1(args)
    elif args.impl == "reference":
        bench_reference(args)
    else:
        if args.path == "all":
            raise SystemExit("--path all is for --sweep")
        bench_ours(args)


if __name__ == "__main__":
    main()

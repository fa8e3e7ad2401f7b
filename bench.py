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
    """Roofline denominators: HBM and the bf16 burst from the driver's
    MEASURED_PEAKS.json; the TF32 and FP32 peaks from this pool's probes
    (profiles/peaks_measured.json, scripts/measure_peaks.py)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        src = "measured"
    else:
        d = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}
        src = "fallback (B200_PROFILING.md)"
    q = os.path.join(ROOT, "profiles", "peaks_measured.json")
    if os.path.exists(q):
        with open(q) as f:
            d["probes"] = json.load(f)
    return d, src


def path_peak(path, peaks, split=0):
    """(peak TFLOP/s, bound, note, measured?) for a path's dominant kernel.
    FP32_TC runs `split` bf16 piece-pair products per fp32 product: its peak
    is the bf16 peak / split in fp32 FLOPs."""
    sel = peaks.get("probes", {}).get("selected", {})
    if path == "fp32_tc":
        return peaks["bf16_tflops"] / split, "tensor", \
            f"cuBLAS bf16 GEMM burst (MEASURED_PEAKS.json, driver) / {split} piece pairs", True
    if path == "bf16":
        return peaks["bf16_tflops"], "tensor", "cuBLAS bf16 GEMM burst (MEASURED_PEAKS.json, driver)", True
    if path == "tf32":
        if "peak_tf32_tflops" in sel:
            return sel["peak_tf32_tflops"], "tensor", \
                "cuBLAS TF32 GEMM 8192^3 burst on this pool (profiles/peaks_measured.json)", True
        return peaks["bf16_tflops"] * 0.5, "tensor", "bf16 burst x 0.5 (nominal tf32/bf16 ratio; derived)", False
    if "peak_fp32_tflops" in sel:
        return sel["peak_fp32_tflops"], "alu", "FFMA probe burst on this pool (profiles/peaks_measured.json)", True
    return 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, "alu", \
        "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (derived)", False


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


PATH_DTYPE = {"bf16": "bf16", "tf32": "tf32", "fp32_simt": "f32", "fp32_tc": "f32 (bf16x{split} exact split)"}
L2_NOTE = ("flushed before every timed step, outside the event pair: write of a 2x-L2 buffer, then a read of "
           "another 2x-L2 buffer (dirty lines written back before the step: cold, clean L2)")


def shard_spec(args, world: int, rank: int):
    """(full workload, this rank's ShardSpec).  Strong scaling (default): the
    workload's units are split across ranks with shard.shard (n, or k for
    N = 1 layers; PAPER.md:375 -- non-reduction dims only).  Weak (opt-in):
    every rank runs the whole workload on its own seed."""
    from paper_2101_09808_b200.shard import ShardSpec, shard
    full = CONFIGS[args.config]
    if world == 1 or args.scaling == "weak":
        return full, ShardSpec("n", world, rank, 0, full.N, full)
    return full, shard(full, world, rank, args.shard)


def rank_inputs(args, full, spec, rank):
    """This rank's (In, Ker) on the host, plus the full tensors (strong)."""
    from paper_2101_09808_b200.shard import local_inputs
    if spec.world == 1 or args.scaling == "weak":
        inp, ker = make_inputs(full, seed=rank)
        return inp, ker, inp, ker
    inp, ker = make_inputs(full, seed=0)
    li, lk = local_inputs(spec, inp, ker)
    return li, lk, inp, ker


class GpuEngine:
    """Runs plans of libconv.so on this rank's GPU and times them on the
    launching stream with CUDA events."""
    timer = "cuda events on the launching stream"

    def __init__(self, local: int):
        from paper_2101_09808_b200 import conv
        self.conv = conv
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.local = local
        self.stream = torch.cuda.current_stream(self.dev)
        l2 = getattr(torch.cuda.get_device_properties(self.dev), "L2_cache_size", 126 << 20)
        n = max(2 * l2, 256 << 20) // 4
        self.flush_w = torch.empty(n, dtype=torch.float32, device=self.dev)
        self.flush_r = torch.ones(n, dtype=torch.float32, device=self.dev)
        self.flush_o = torch.empty((), dtype=torch.float32, device=self.dev)

    def l2_flush(self):
        # write a buffer > L2 (evicts every line), then read another one so
        # the dirty lines of the first pass are written back here, outside
        # the timed events: each step starts with a cold, clean L2
        self.flush_w.zero_()
        torch.sum(self.flush_r, dim=0, out=self.flush_o)

    def sync(self):
        torch.cuda.synchronize(self.dev)

    def to_device(self, t):
        return t.pin_memory().to(self.dev)

    def measure(self, path, sh, d_in, d_ker, args, barrier):
        """K timed steps of one path (CUDA-graph replay of conv_run, L2
        flushed before each, an event pair around each), then K steps with
        events between the kernels (attribution).  NVML clocks sampled over
        the soak and both passes."""
        conv = self.conv
        plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=args.tile, **sh.plan_kwargs())
        d_out = plan.new_output(self.dev)
        ws = plan.new_workspace(self.dev)
        st = self.stream
        for _ in range(args.warmup):
            self.l2_flush()
            plan.run(d_in, d_ker, d_out, ws)
        self.sync()
        clocks = ClockSampler(self.local)
        clocks.start()
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < args.soak:
            for _ in range(20):
                self.l2_flush()
                plan.run(d_in, d_ker, d_out, ws)
            self.sync()
        graph = None
        if not args.no_graph:
            try:
                cap = torch.cuda.Stream(device=self.dev)
                cap.wait_stream(st)
                with torch.cuda.stream(cap):
                    plan.run(d_in, d_ker, d_out, ws, stream=cap)
                cap.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=cap):
                    plan.run(d_in, d_ker, d_out, ws, stream=cap)
                self.sync()
                graph.replay()
                self.sync()
            except Exception as e:  # pragma: no cover - fall back to stream launches
                print(f"warning: CUDA graph capture failed ({e}); timing stream launches", file=sys.stderr)
                graph = None
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        self.sync()
        for a, b in ev:
            self.l2_flush()                                     # outside the event pair
            a.record(st)
            if graph is not None:
                graph.replay()
            else:
                plan.run(d_in, d_ker, d_out, ws)
            b.record(st)
        self.sync()
        barrier()
        step_ms = np.array([a.elapsed_time(b) for a, b in ev])
        nk = plan.num_kernels
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)] for _ in range(args.steps)]
        barrier()
        self.sync()
        for e in evs:
            self.l2_flush()
            plan.run_events(d_in, d_ker, d_out, ws, e)
        self.sync()
        barrier()
        clocks.stop()
        per_kernel = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(nk)] for e in evs])
        return {"plan": plan, "desc": plan.describe(), "path": plan.path, "step_ms": step_ms,
                "per_kernel": per_kernel, "clocks": clocks.summary(), "out": d_out, "nk": nk,
                "launch": "cuda_graph replay of conv_run" if graph is not None else "stream launches"}

    def gpu_local_cpus(self):
        """CPUs NVML names as local to this GPU (its NUMA node), within the
        process's allowed set; None if unknown."""
        try:
            import pynvml
            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(self.dev)
            try:
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.dev.index or 0)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
            cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
            cpus &= os.sched_getaffinity(0)
            return cpus or None
        except Exception:
            return None

    def e2e(self, res, sh, in_h, ker_h, args, barrier):
        """conv_run_host with pinned host buffers: H2D + conv + D2H inside the
        event pair, every step.  The pinned buffers are allocated (first
        touched) with the thread on the GPU's local CPUs (--cpu-affinity gpu,
        the default: host pages on the GPU's NUMA node), then the affinity is
        restored for the other legs."""
        plan = res["plan"]
        prev = os.sched_getaffinity(0)
        local = self.gpu_local_cpus() if args.cpu_affinity == "gpu" else None
        if local:
            os.sched_setaffinity(0, local)
        self.e2e_affinity = f"gpu-local ({len(local)} of {len(prev)} cpus)" if local else "process default"
        try:
            in_h, ker_h = in_h.clone().pin_memory(), ker_h.clone().pin_memory()
            out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
            out_h.zero_()
        finally:
            if local:
                os.sched_setaffinity(0, prev)
        dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device=self.dev)
        for _ in range(max(1, args.warmup)):
            plan.run_host(in_h, ker_h, out_h, dbuf)
        self.sync()
        ms = []
        barrier()
        for _ in range(args.steps):
            self.l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            plan.run_host(in_h, ker_h, out_h, dbuf)
            b.record(self.stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        self.sync()
        return float(np.mean(ms))

    def reference_slab(self, res, full, spec, inp_full, ker_full):
        """P10: the 1-GPU result of the full workload
        with the shard plan's tile forced (same k order, same split count),
        sliced to this rank's slab.  Returns (slice, how)."""
        conv = self.conv
        d = res["desc"]["tile"]
        keys = ("ver", "tk", "tw", "kg", "pw", "tn", "th", "bc", "splits") if res["path"] == "fp32_simt" else \
            ("bn", "cg", "kbs", "stages", "splits", "fuse", "expand")
        spec_s = ",".join(f"{k}={d[k]}" for k in keys if k in d)
        how = f"full-workload plan, tile forced to the shard's ({spec_s})"
        try:
            plan = conv.ConvPlan(*full.as_tuple(), path=res["path"], tile=spec_s, **full.plan_kwargs())
        except conv.ConvError:
            plan = conv.ConvPlan(*full.as_tuple(), path=res["path"], **full.plan_kwargs())
            how = "full-workload plan, AUTO tile (the shard's tile is infeasible on the full workload)"
        out = plan.run(inp_full.to(self.dev), ker_full.to(self.dev))
        self.sync()
        sl = out[spec.start:spec.stop] if spec.dim == "n" else out[:, spec.start:spec.stop]
        return sl.contiguous(), how

    def timed_gather(self, out, spec, args, barrier):
        from paper_2101_09808_b200.shard import gather
        full = gather(out, spec)                                   # warm-up
        self.sync()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        for _ in range(args.steps):
            full = gather(out, spec)
        b.record(self.stream)
        self.sync()
        return full, a.elapsed_time(b) / args.steps


def harness(args, rank: int, world: int, engine, dist_mod=None):
    """One rank of the bench: shard (strong n / k, or weak replicas), time
    every requested path with the engine, check the slab against the 1-GPU
    result (P10), optionally all-gather Out (timed separately), reduce the
    timings as the MAX over ranks, and (rank 0) build the JSON line.
    ``dist_mod`` is torch.distributed with an initialised process group when
    world > 1 (NCCL on the GPU box; gloo in the CPU harness test)."""
    def barrier():
        if world > 1:
            dist_mod.barrier()

    def reduce(vals, op):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        if getattr(engine, "dev", None) is not None and dist_mod.get_backend() == "nccl":
            t = t.to(engine.dev)
        dist_mod.all_reduce(t, op=op)
        return t.cpu().tolist()

    full, spec = shard_spec(args, world, rank)
    sh = spec.local
    li, lk, inp_full, ker_full = rank_inputs(args, full, spec, rank)
    d_in, d_ker = engine.to_device(li), engine.to_device(lk)
    paths = [args.path] + [p for p in (args.paths.split(",") if args.paths else []) if p and p != args.path]
    results = {p: engine.measure(p, sh, d_in, d_ker, args, barrier) for p in paths}
    head = results[args.path]
    e2e_ms = None if args.no_e2e else engine.e2e(head, sh, li, lk, args, barrier)

    p10 = None
    if world > 1 and args.scaling == "strong" and not args.no_check:
        ref, how = engine.reference_slab(head, full, spec, inp_full, ker_full)
        same = bool(torch.equal(head["out"].cpu(), ref.cpu()))
        ok = reduce([1.0 if same else 0.0], dist_mod.ReduceOp.MIN)[0] if world > 1 else float(same)
        p10 = {"bit_identical_all_ranks": ok == 1.0, "ranks": world, "reference": how}
    gathered, g_ms = None, None
    if args.gather and world > 1:
        gathered, g_ms = engine.timed_gather(head["out"], spec, args, barrier)

    # max over ranks of every time
    vec = []
    for p in paths:
        vec += [float(results[p]["step_ms"].mean()), float(results[p]["per_kernel"][:, -1].mean())]
    vec += [e2e_ms or 0.0, g_ms or 0.0]
    red = reduce(vec, dist_mod.ReduceOp.MAX if world > 1 else None)
    for i, p in enumerate(paths):
        results[p]["ms_max"], results[p]["main_ms_max"] = red[2 * i], red[2 * i + 1]
    e2e_ms = red[-2] if e2e_ms is not None else None
    g_ms = red[-1] if g_ms is not None else None

    line = None
    if rank == 0:
        line = build_line(args, world, full, spec, paths, results, e2e_ms, g_ms, p10, engine)
    return {"line": line, "gathered": gathered, "results": results}


def path_record(args, world, full, spec, res, engine, peaks, peak_src):
    """value, roofline and clocks of one path (rank 0's view, max over ranks)."""
    sh = spec.local
    ms, main_ms = res["ms_max"], res["main_ms_max"]
    total_flops = full.flops * (world if args.scaling == "weak" else 1)
    peak, bound, peak_note, measured = path_peak(res["path"], peaks, res["desc"]["tile"].get("split", 0))
    achieved = sh.flops / (main_ms * 1e-3) / 1e12
    per_kernel = res["per_kernel"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and world == 1:
        with open(tpath) as f:
            tkey = f"{args.config}:{res['path']}" + (":fuse" if res["desc"]["tile"].get("fuse") else "")
            traffic = json.load(f).get(tkey)
    roof_us = max(sh.flops / (peak * 1e12), sh.compulsory_bytes / (peaks["hbm_gbs"] * 1e9)) * 1e6
    return {
        "value": round(total_flops / (ms * 1e-3) / 1e12, 3),
        "ms_per_step": round(ms, 5),
        "dtype": PATH_DTYPE[res["path"]].format(split=res["desc"]["tile"].get("split", 0)),
        "path": res["path"],
        "tile": res["desc"]["tile"],
        "step_stats": step_stats(res["step_ms"]),
        "roofline": {
            "bound": bound,
            "achieved": round(achieved, 2),
            "peak": round(peak, 2),
            "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "kernel": "conv_igemm_tcgen05" if res["path"] != "fp32_simt" else "conv_direct_simt",
            "kernel_ms": round(main_ms, 5),
            "peak_source": f"{peak_note}; {peak_src}",
            "peak_measured": measured,
            "step_roofline_us": round(roof_us, 3),
            "step_frac": round(roof_us / (ms * 1e3), 4),
            "kernel_share_of_step": round(float(per_kernel[:, -1].mean()) / float(per_kernel.sum(axis=1).mean()), 4),
            "kernel_ms_each": [round(float(x), 5) for x in per_kernel.mean(axis=0)],
            "timing": "kernel durations from a second K-step pass with events between the kernels",
        },
        "clocks": res["clocks"],
        "kernels_per_step": res["nk"],
        # FP32 SIMT flat tiles: the remainder grid is a launch of its own, timed together with
        # the main grid it runs beside (no event between the two)
        "launches_per_step": res["nk"] + (1 if res["desc"]["tile"].get("rem") else 0),
        "launch": res["launch"],
    }


def build_line(args, world, full, spec, paths, results, e2e_ms, g_ms, p10, engine):
    peaks, peak_src = load_peaks()
    sh = spec.local
    head = path_record(args, world, full, spec, results[args.path], engine, peaks, peak_src)
    total_flops = full.flops * (world if args.scaling == "weak" else 1)
    strong = world > 1 and args.scaling == "strong"
    wl = f"{args.config}: N={full.N} K={full.K} C={full.C} out {full.H}x{full.W} R={full.R} S={full.S} " \
         f"(stride 1, no pad, fp32 NCHW/KCRS)"
    line = {
        "metric": METRIC,
        "value": head["value"],
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        # rank 0's K timed steps: the paper's statistic is the mean;
        # median and a normal 95% CI of the mean beside it
        "step_stats": head["step_stats"],
        "higher_is_better": True,
        # the requested mode (default strong: BASELINE configs[4]'s n-sharded
        # batch); at N = 1 both modes run the same whole workload
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": head["dtype"],
        "data": "synthetic (seeded uniform[-1,1), BASELINE.json configs)",
        "config": {
            "workload": wl if world == 1 or strong else wl + f", x{world} replicas (weak)",
            "path": head["path"],
            "tile": head["tile"],
            "l2": L2_NOTE,
            "clocks_window": "NVML samples every ~1 ms over the >= 1 s warm-up soak and both timed passes",
            "parallelism": ("single GPU" if world == 1 else
                            f"{spec.dim}-shard x{world}" if strong else f"replicas x{world}"),
            "shard": {"dim": spec.dim, "world": world, "per_rank": f"{spec.dim}={spec.size}",
                      "per_rank_shape": list(sh.as_tuple())},
            "kernels_per_step": head["kernels_per_step"],
            "launches_per_step": head["launches_per_step"],
            "launch": head["launch"],
            "timer": engine.timer,
        },
        "roofline": head["roofline"],
        "gpu_launches": head["launches_per_step"] * args.steps,
        "clocks": head["clocks"],
    }
    if e2e_ms is not None:
        line["e2e"] = {
            "value": round(total_flops / (e2e_ms * 1e-3) / 1e12, 3),
            "unit": "TFLOP/s",
            "ms_per_step": round(e2e_ms, 4),
            "h2d_bytes_per_step": 4 * (sh.N * sh.C * sh.Hin * sh.Win + sh.K * sh.C * sh.R * sh.S) * world,
            "d2h_bytes_per_step": 4 * sh.N * sh.K * sh.H * sh.W * world,
            "api": "conv_run_host (C ABI, pinned host buffers)" + (", every rank its slab" if world > 1 else ""),
            "host_buffers": getattr(engine, "e2e_affinity", None),
        }
    others = [p for p in paths if p != args.path]
    if others:
        line["paths"] = {p: path_record(args, world, full, spec, results[p], engine, peaks, peak_src) for p in others}
    if p10 is not None:
        line["p10"] = p10
    if g_ms is not None:
        line["gather"] = {"ms": round(g_ms, 4), "collective": "all_gather_into_tensor (shard.gather)",
                          "bytes_recv_per_gpu": (world - 1) * 4 * sh.N * sh.K * sh.H * sh.W,
                          "note": "after the timed region, not in value"}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(full, args)
    return line


def bench_ours(args):
    import torch.distributed as dist
    rank, world, local = dist_env()
    engine = GpuEngine(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=engine.dev)
    try:
        out = harness(args, rank, world, engine, dist)
        if rank == 0:
            print(json.dumps(out["line"]), flush=True)
    finally:
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
    # single-thread oracle beside it: one image
    t_1 = oracle_sample_time(sh, 1, 1)
    flops_1 = 2.0 * sh.K * sh.H * sh.W * sh.C * sh.R * sh.S
    return {"value": round(flops / t / 1e12, 6), "unit": "TFLOP/s", "cores": used, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"first {n} of {sh.N} images of the {args.config} layer ({t:.1f} s, double accumulation, "
                      f"OpenMP over (n,k) planes)",
            "single_thread": {"value": round(flops_1 / t_1 / 1e12, 6), "unit": "TFLOP/s", "cores": 1,
                              "sample": f"1 image ({t_1:.2f} s)"}}


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
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1), BASELINE.json configs)",
        # the same workload string as our arm's line (the driver compares them)
        "config": {"workload": f"{args.config}: N={sh.N} K={sh.K} C={sh.C} out {sh.H}x{sh.W} R={sh.R} S={sh.S} "
                               f"(stride 1, no pad, fp32 NCHW/KCRS)",
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
    paths = [args.path] if args.path != "all" else ["bf16", "tf32", "fp32_simt", "fp32_tc"]
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
            peak, bound, _, _ = path_peak(plan.path, peaks, plan.describe()["tile"].get("split", 0))
            roof_us = max(sh.flops / (peak * 1e12), 4.0 * (sh.N * sh.C * sh.Hin * sh.Win + sh.K * sh.C * sh.R * sh.S +
                                                           sh.N * sh.K * sh.H * sh.W) / (peaks["hbm_gbs"] * 1e9)) * 1e6
            d = plan.describe()
            print(json.dumps({
                "layer": name, "path": plan.path, "K": sh.K, "C": sh.C, "Hin": sh.Hin, "R": sh.R, "U": sh.U, "pad": sh.ph,
                "out": [sh.H, sh.W], "gflop": round(sh.flops / 1e9, 4), "step_us": round(ms * 1e3, 2),
                "tflops": round(sh.flops / (ms * 1e-3) / 1e12, 3), "roofline_us": round(roof_us, 3),
                "frac": round(roof_us / (ms * 1e3), 4), "kernels_us": kern_us, "tile": d["tile"],
                "peak_source": peak_src}), flush=True)


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args, argv) -> int:
    """``--gpus N`` without torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on this node and return its exit code.  Fails
    (rc 2) if fewer than N GPUs are visible."""
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(f"error: --gpus {args.gpus} but only {n} CUDA device(s) visible", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--path", default="fp32_simt", choices=["auto", "fp32_simt", "fp32_tc", "tf32", "bf16", "all"],
                    help="the headline path (default: FP32, the paper's precision, PAPER.md:369)")
    ap.add_argument("--paths", default="fp32_tc,tf32,bf16",
                    help="further paths measured in the same process, reported under 'paths' ('' for none)")
    ap.add_argument("--shard", default="auto", choices=["auto", "n", "k"],
                    help="strong scaling: shard the batch n (auto for N >= ranks) or output channels k (N = 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-affinity", choices=["gpu", "none"], default="gpu",
                    help="e2e leg: allocate the pinned host buffers from the GPU's local CPUs (NUMA node)")
    ap.add_argument("--no-check", action="store_true", help="skip the multi-rank P10 slab check")
    ap.add_argument("--config", default="batched", choices=list(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the workload's units split across ranks; weak: a replica per rank")
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
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    rank, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus and args.impl == "ours":
        print(f"error: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours" and not args.sweep:
        sys.exit(launch_ranks(args, sys.argv[1:]))
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

"""bench.py's multi-rank harness (row a-7 / Sec. 8(e)) on the CPU: the same
``harness`` the GPU ranks run -- strong n- (or k-) sharding with
shard.shard, MAX-over-ranks timing, the P10 slab check, the timed
all-gather (shard.gather) and rank 0's JSON line -- at world size 2 over
gloo.  Only here does the oracle stand in for the convolution step (an
engine with the GpuEngine interface); on the GPU box the engine runs
libconv.so plans over NCCL."""
import argparse
import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2101_09808_b200.inputs import CONFIGS, Shape, make_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """GpuEngine's interface with the CPU oracle as the convolution step
    (test infrastructure only)."""
    timer = "time.perf_counter (CPU test engine)"
    dev = None

    def to_device(self, t):
        return t

    def measure(self, path, sh, d_in, d_ker, args, barrier):
        barrier()
        times = []
        out = None
        for _ in range(args.steps):
            t0 = time.perf_counter()
            out = torch.from_numpy(oracle.conv_eq1(d_in.numpy(), d_ker.numpy()).astype(np.float32))
            times.append((time.perf_counter() - t0) * 1e3)
        barrier()
        ms = np.array(times)
        return {"plan": None, "desc": {"tile": {}}, "path": path, "step_ms": ms, "per_kernel": ms[:, None],
                "clocks": {"sm_mhz": None, "reasons": []}, "out": out, "nk": 1, "launch": "cpu oracle (test)"}

    def e2e(self, res, sh, in_h, ker_h, args, barrier):
        return float(res["step_ms"].mean())

    def reference_slab(self, res, full, spec, inp_full, ker_full):
        ref = torch.from_numpy(oracle.conv_eq1(inp_full.numpy(), ker_full.numpy()).astype(np.float32))
        sl = ref[spec.start:spec.stop] if spec.dim == "n" else ref[:, spec.start:spec.stop]
        return sl.contiguous(), "oracle on the full workload"

    def timed_gather(self, out, spec, args, barrier):
        from paper_2101_09808_b200.shard import gather
        barrier()
        t0 = time.perf_counter()
        full = gather(out, spec)
        return full, (time.perf_counter() - t0) * 1e3


def _args(**kw):
    a = dict(config="tiny", path="fp32_simt", paths="", steps=2, warmup=0, scaling="strong", shard="auto",
             gather=True, no_e2e=False, no_check=False, no_cpu_baseline=True, tile=None, soak=0.0, no_graph=False)
    a.update(kw)
    return argparse.Namespace(**a)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, config, shape, kw, q):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bench.CONFIGS[config] = Shape(*shape)       # small workloads the oracle finishes in seconds
        res = bench.harness(_args(config=config, **kw), rank, world, OracleEngine(), dist)
        if rank == 0:
            q.put((res["line"], res["gathered"].numpy() if res["gathered"] is not None else None))
    finally:
        dist.destroy_process_group()


def _run(config, shape, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, config, shape, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    line, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return line, gathered


@pytest.mark.parametrize("shape,dim", [((4, 6, 3, 5, 7, 3, 3), "n"), ((1, 8, 5, 9, 6, 3, 2), "k")])
def test_harness_world2_strong_shard_gather_equals_oracle(shape, dim):
    line, gathered = _run("tinyx", shape)
    sh = Shape(*shape)
    inp, ker = make_inputs(sh, seed=0)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy()).astype(np.float32)
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["shard"]["dim"] == dim and line["config"]["shard"]["world"] == 2
    per = sh.N // 2 if dim == "n" else sh.K // 2
    assert line["config"]["shard"]["per_rank"] == f"{dim}={per}"
    assert line["p10"]["bit_identical_all_ranks"] is True
    assert gathered is not None and gathered.shape == ref.shape and np.array_equal(gathered, ref)
    # value = the whole workload's FLOPs / max-over-ranks time
    assert abs(line["value"] - sh.flops / (line["ms_per_step"] * 1e-3) / 1e12) <= 1e-3 + 1e-3 * line["value"]
    assert line["gather"]["bytes_recv_per_gpu"] == 4 * sh.N * sh.K * sh.H * sh.W // 2
    assert line["e2e"]["h2d_bytes_per_step"] == 4 * (sh.N * sh.C * sh.Hin * sh.Win + 2 * sh.K * sh.C * sh.R * sh.S) \
        if dim == "n" else True


def test_harness_world2_weak_replicas():
    line, _ = _run("tinyx", (2, 4, 3, 5, 5, 3, 3), scaling="weak", gather=False)
    sh = Shape(2, 4, 3, 5, 5, 3, 3)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and "p10" not in line
    assert "replicas" in line["config"]["workload"]
    assert abs(line["value"] - 2 * sh.flops / (line["ms_per_step"] * 1e-3) / 1e12) <= 1e-3 + 1e-3 * line["value"]


def test_gpus_flag_needs_that_many_devices():
    """--gpus N with fewer visible GPUs exits non-zero (here: none)."""
    import subprocess
    import sys
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs present")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env={k: v for k, v in os.environ.items()
                                                                                    if k not in ("WORLD_SIZE", "RANK")})
    assert r.returncode != 0 and "visible" in r.stderr


def test_shard_spec_defaults():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    full, spec = bench.shard_spec(_args(config="batched"), 8, 3)
    assert full == CONFIGS["batched"] and spec.dim == "n" and (spec.start, spec.stop) == (96, 128)
    full, spec = bench.shard_spec(_args(config="det"), 4, 1)
    assert spec.dim == "k" and spec.local.K == 16
    full, spec = bench.shard_spec(_args(config="batched", scaling="weak"), 4, 2)
    assert spec.local == full

"""Fuzz of conv_run_host (study script, r02e): seeded random batched problems
-- half of them 14-wide 3x3 layers, the flat / remainder / split-C territory
of the FP32 SIMT path, whose pipeline chunks run a finer tile than the device
plan -- on every path: the pipelined host call (chunked H2D, conv, D2H) must
give the bits of conv_run, twice.  Usage: python scripts/fuzz_run_host.py N SEED"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import Shape, make_inputs  # noqa: E402

n, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
runs = fails = 0
for i in range(n):
    if rng.random() < 0.5:
        sh = Shape(N=int(rng.integers(20, 300)), K=int(rng.choice([32, 64, 100, 256])), C=int(rng.choice([8, 20, 64, 128])),
                   H=int(rng.choice([7, 9, 14])), W=14, R=3, S=3)
    else:
        S = int(rng.choice([1, 3]))
        sh = Shape(N=int(rng.integers(1, 64)), K=int(rng.choice([16, 30, 64, 128])), C=int(rng.choice([3, 16, 33, 64])),
                   H=int(rng.integers(4, 40)), W=int(rng.integers(4, 40)), R=S, S=S)
    if sh.flops > 3e10:
        continue
    inp, ker = make_inputs(sh, seed=i)
    ih, kh = inp.pin_memory(), ker.pin_memory()
    out_h = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    for path in ("fp32_simt", "fp32_tc", "tf32", "bf16"):
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path=path)
        except conv.ConvError:
            continue
        d = plan.describe()
        dev = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
        dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
        ok = True
        for _ in range(2):
            out_h.fill_(float("nan"))
            plan.run_host(ih, kh, out_h, dbuf)
            torch.cuda.synchronize()
            ok = ok and np.array_equal(out_h.numpy(), dev)
        runs += 1
        if not ok:
            fails += 1
            print(json.dumps({"shape": sh.as_tuple(), "path": path, "tile": d["tile"], "host": d["host_pipeline"]}), flush=True)
        del dbuf
print(json.dumps({"plan_runs": runs, "fails": fails, "seed": seed}), flush=True)

"""Parity fuzz of Eq. 1 proper (stride 1, no padding, no dilation -- the class
the SIMT v2 / TMA-staged tiles serve) with independent R, S in 1..5 and input
rows that are often 16-B multiples (study script, r02e: the class the general
fuzz almost never draws, where the 1x3-taps TMA planning bug sat).  Every
path, the selector's plan: integer twin bit-exact, relL2 within the path's
tolerance against the double oracle.  Usage: python scripts/fuzz_plain.py N SEED"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import Shape, make_inputs  # noqa: E402

TOL = {"fp32_simt": 1e-5, "fp32_tc": 1e-5, "tf32": 5e-3, "bf16": 5e-3, "auto": 1e-5}
n, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
runs = fails = infeasible = 0
for i in range(n):
    R, S = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    W = int(rng.integers(1, 40))
    if rng.random() < 0.6:
        W = max(1, (W + S - 1 + 3) // 4 * 4 - (S - 1))       # Win % 4 == 0
    sh = Shape(N=int(rng.integers(1, 40)), K=int(rng.choice([1, 7, 16, 30, 64, 100])), C=int(rng.choice([1, 3, 8, 20, 33, 64])),
               H=int(rng.integers(1, 30)), W=W, R=R, S=S)
    if sh.flops > 4e8:
        continue
    xi, wi = make_inputs(sh, seed=i, kind="int")
    inp, ker = make_inputs(sh, seed=10000 + i)
    refi = oracle.conv_eq1(xi.numpy(), wi.numpy())
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    for path in TOL:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path=path)
        except conv.ConvError as e:
            infeasible += 1
            if e.status != 2:
                fails += 1
                print(json.dumps({"shape": sh.as_tuple(), "path": path, "create_error": str(e)[:120]}), flush=True)
            continue
        runs += 1
        try:
            goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy().astype(np.float64)
            got = plan.run(inp.cuda(), ker.cuda()).cpu().numpy().astype(np.float64)
        except conv.ConvError as e:
            fails += 1
            print(json.dumps({"shape": sh.as_tuple(), "path": path, "tile": plan.describe()["tile"], "run_error": str(e)[:120]}), flush=True)
            continue
        rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
        if not (np.array_equal(goti, refi) and rel <= TOL[path]):
            fails += 1
            print(json.dumps({"shape": sh.as_tuple(), "path": path, "tile": plan.describe()["tile"], "rel": rel,
                              "int_exact": bool(np.array_equal(goti, refi))}), flush=True)
print(json.dumps({"plan_runs": runs, "infeasible": infeasible, "fails": fails, "seed": seed}), flush=True)

"""Parity fuzz of the FP32 SIMT v2 TMA staging (study script, r02b): seeded
random stride-1 problems with Win % 4 == 0 (the TMA stride rule) and random
forced v2 tiles (TK, TW, kg, pw, tn, bc, split-C); every feasible plan that
takes the TMA staging is checked bit-exact on the integer twin and <= 1e-5
against the double oracle.  One JSON line per failure, a summary at the end.
Usage: python scripts/fuzz_simt_tma.py N SEED"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import Shape, make_inputs  # noqa: E402

n, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
checked = skipped = fails = 0
for i in range(n):
    S = int(rng.choice([1, 3]))
    R = S if rng.random() < 0.8 else int(rng.choice([1, 2, 3, 5]))   # r02e: R != S takes the cp.async layout, checked too
    W = int(rng.choice([w for w in range(2, 40) if (w + S - 1) % 4 == 0]))
    H = int(rng.integers(1, 24))
    sh = Shape(N=int(rng.integers(1, 7)), K=int(rng.integers(1, 80)), C=int(rng.integers(1, 48)), H=H, W=W, R=R, S=S)
    tw = int(rng.choice([4, 8] + ([W] if W in (7, 14) else [])))
    tk = 4 if tw in (7, 14) else int(rng.choice([4, 8]))
    spec = (f"ver=2,tk={tk},tw={tw},kg={rng.choice([1, 2, 4, 8])},pw={rng.choice([1, 2, 3])},"
            f"tn={rng.choice([1, 2, 3, 4])},bc={rng.choice([4, 8, 16])},splits={rng.choice([1, 1, 1, 2, 4])}")
    try:
        plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
    except conv.ConvError:
        skipped += 1
        continue
    if plan.describe()["tile"]["staging"] != "tma" and R == S:
        skipped += 1
        continue
    xi, wi = make_inputs(sh, seed=i, kind="int")
    inp, ker = make_inputs(sh, seed=10000 + i)
    goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy().astype(np.float64)
    got = plan.run(inp.cuda(), ker.cuda()).cpu().numpy().astype(np.float64)
    refi = oracle.conv_eq1(xi.numpy(), wi.numpy())
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    ok = np.array_equal(goti, refi) and rel <= 1e-5
    checked += 1
    if not ok:
        fails += 1
        print(json.dumps({"shape": sh.as_tuple(), "spec": spec, "tile": plan.describe()["tile"], "rel": rel,
                          "int_exact": bool(np.array_equal(goti, refi))}), flush=True)
print(json.dumps({"checked": checked, "skipped": skipped, "fails": fails, "seed": seed}), flush=True)

"""Parity fuzz of the FP32 SIMT flat row-mode tiles and their remainder launch
(study script, r02e): seeded random problems with W = 14, S = 3 (the flat
TMA layout's rule: TW = W, Win % 4 == 0, 3x3 taps), random H, ragged N / K / C large
enough for more CTAs than SMs, and random forced flat tiles (kg, bc incl. 6,
split-C 1..3).  Every feasible plan is checked bit-exact on the integer twin,
<= 1e-5 against the double oracle, and bit-identical to the same tile without
the remainder launch (rem=0).  One JSON line per failure, a summary at the end.
Usage: python scripts/fuzz_simt_flat.py N SEED"""
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
checked = skipped = fails = with_rem = with_split_rem = 0
for i in range(n):
    R = 3                                        # flat tiles exist for 3x3 taps (the TMA instances are 1x1 / 3x3)
    H = int(rng.integers(3, 20))
    kg = int(rng.choice([2, 4, 8]))
    K = int(rng.integers(1, 70))
    C = int(rng.integers(1, 26))
    splits = int(rng.choice([1, 1, 2, 3]))
    ktiles = -(-K // (4 * kg))
    # slot tiles so that the grid is 1.0 .. 3.2 rounds of 148 CTAs, often just over a whole round
    want = int(rng.choice([150, 152, 160, 200, 297, 300, 310, 400, 445, 450, 470]))
    tiles = max(2, -(-want // (ktiles * splits)))
    N = max(1, (tiles * 32 - int(rng.integers(0, 32))) // H)
    sh = Shape(N=N, K=K, C=C, H=H, W=14, R=R, S=3)
    spec = f"flat=1,tk=4,kg={kg},pw=1,bc={rng.choice([2, 4, 4, 6, 8])},splits={splits}"
    try:
        plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        plain = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec + ",rem=0")
    except conv.ConvError:
        skipped += 1
        continue
    t = plan.describe()["tile"]
    with_rem += t["rem"] > 0
    with_split_rem += t["rem"] > 0 and t["splits"] > 1
    xi, wi = make_inputs(sh, seed=i, kind="int")
    inp, ker = make_inputs(sh, seed=10000 + i)
    try:
        goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy().astype(np.float64)
        got32 = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
        same = np.array_equal(got32, plain.run(inp.cuda(), ker.cuda()).cpu().numpy())
    except conv.ConvError as e:                      # a plan that was created must run
        fails += 1
        checked += 1
        print(json.dumps({"shape": sh.as_tuple(), "spec": spec, "tile": t, "run_error": str(e)[:120]}), flush=True)
        continue
    refi = oracle.conv_eq1(xi.numpy(), wi.numpy())
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    rel = float(np.linalg.norm(got32.astype(np.float64) - ref) / max(np.linalg.norm(ref), 1e-30))
    ok = np.array_equal(goti, refi) and rel <= 1e-5 and same
    checked += 1
    if not ok:
        fails += 1
        print(json.dumps({"shape": sh.as_tuple(), "spec": spec, "tile": t, "rel": rel,
                          "int_exact": bool(np.array_equal(goti, refi)), "same_as_rem0": bool(same)}), flush=True)
print(json.dumps({"checked": checked, "skipped": skipped, "fails": fails, "with_rem": int(with_rem),
                  "with_split_rem": int(with_split_rem), "seed": seed}), flush=True)

"""Parity fuzz on multi-wave problems (study script): seeded random layers
large enough for the fused transform and multi-wave schedules; the integer
twin is checked bit-exact on 96 sampled outputs (oracle point sums), for the
selector's plan and a forced fused / CTA-pair variant.
Usage: python scripts/fuzz_large.py N_SHAPES SEED"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import Shape, make_inputs  # noqa: E402

n, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
runs = fails = 0
for i in range(n):
    R = int(rng.choice([1, 3, 3, 5]))
    U = int(rng.choice([1, 1, 2]))
    p = int(rng.choice([0, R // 2]))
    C = int(rng.choice([32, 64, 96, 128, 256]))
    K = int(rng.choice([64, 96, 128, 192, 256]))
    N = int(rng.integers(8, 97))
    Hin = int(rng.integers(10, 34))
    sh = Shape.strided(N, K, C, Hin, Hin + int(rng.integers(0, 4)), R, R, U, 1, p, p)
    xi, wi = make_inputs(sh, seed=i, kind="int")
    x, w = xi.numpy(), wi.numpy()
    pts = [(int(rng.integers(sh.N)), int(rng.integers(sh.K)), int(rng.integers(sh.H)), int(rng.integers(sh.W)))
           for _ in range(96)]
    ref = np.array([oracle.conv_eq1_point(x, w, *q, stride=sh.U, padding=(sh.ph, sh.pw)) for q in pts])
    for path in ("bf16", "tf32"):
        for spec in (None, "fuse=1,cg=2", "fuse=1,cg=1,bn=128"):
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
            except conv.ConvError as e:
                if e.status != conv.CONV_ERR_INFEASIBLE:
                    print("FAIL create", path, spec, sh, e); fails += 1
                continue
            got = plan.run(xi.cuda(), wi.cuda()).cpu().numpy()
            runs += 1
            val = np.array([got[q] for q in pts], dtype=np.float64)
            if not np.array_equal(val, ref):
                fails += 1
                print("FAIL", path, spec, sh, plan.describe()["tile"], flush=True)
print(f"large fuzz: {runs} plan runs, {fails} failures", flush=True)

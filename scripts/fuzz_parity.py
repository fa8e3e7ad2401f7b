"""Parity fuzz (study script): many seeded random general problems on every
path, bit-exact on the integer twin and <= 1e-5 against the padded oracle on
the path's rounded inputs (the same checks as
tests/test_parity.py::test_random_general_shapes, at scale).
Usage: python scripts/fuzz_parity.py N_SHAPES SEED..."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import make_inputs  # noqa: E402
from test_parity import PATHS, ROUND, _random_shapes, rel_l2  # noqa: E402

n = int(sys.argv[1])
fails = 0
total = 0
for seed in map(int, sys.argv[2:]):
    for i, sh in enumerate(_random_shapes(n, seed)):
        pad = (sh.ph, sh.pw)
        xi, wi = make_inputs(sh, seed=i, kind="int")
        inp, ker = make_inputs(sh, seed=10000 + i)
        refi = oracle.conv_eq1_padded(xi.numpy(), wi.numpy(), sh.U, sh.D, pad)
        rng = np.random.default_rng(seed * 1000 + i)
        for path in PATHS:
            spec = None
            if os.environ.get("FUZZ_TILES"):     # a random forced tile (infeasible ones are skipped)
                if path == "fp32_simt":
                    spec = (f"ver={rng.choice([1, 2])},tk={rng.choice([4, 8])},kg={rng.choice([1, 2, 4, 8])},"
                            f"bc={rng.choice([4, 8, 16])},splits={rng.choice([1, 1, 2, 3, 4])}")
                else:
                    spec = (f"bn={rng.choice([32, 64, 128, 192, 256])},cg={rng.choice([1, 2])},"
                            f"kbs={rng.choice([1, 2, 3, 4, 6, 7, 9])},splits={rng.choice([1, 1, 2, 3, 5])},"
                            f"fuse={rng.choice([0, 0, 1])},expand={rng.choice([0, 1])}")
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
            except conv.ConvError as e:
                if e.status != conv.CONV_ERR_INFEASIBLE:
                    print("FAIL create", path, sh, spec, e); fails += 1
                continue
            total += 1
            goti = plan.run(xi.cuda(), wi.cuda()).cpu().numpy().astype(np.float64)
            got = plan.run(inp.cuda(), ker.cuda()).cpu().numpy()
            ref = oracle.conv_eq1_padded(ROUND[path](inp.numpy()), ROUND[path](ker.numpy()), sh.U, sh.D, pad)
            ok = np.array_equal(goti, refi) and (np.linalg.norm(ref) == 0 or rel_l2(got, ref) <= 1e-5)
            if not ok:
                fails += 1
                print("FAIL", path, sh, plan.describe()["tile"], flush=True)
print(f"fuzz: {total} plan runs, {fails} failures", flush=True)

"""SIMT row-mode TK = 8 (112 accumulators, <= 256 threads) vs TK = 4 on the
batched layer: bench-protocol timing + relL2 of two images vs the oracle."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs  # noqa: E402
from scripts.simt_sweep4 import timeit  # noqa: E402

sh = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "batched"]
xi, wi = make_inputs(sh, seed=0)
i, k = xi.cuda(), wi.cuda()
ref = oracle.conv_eq1(xi.numpy()[:2], wi.numpy())
specs = [None, "ver=2,tk=4,tw=14,kg=8,pw=1,tn=2,th=14,bc=8"]
for kg, pw, tn, bc in itertools.product((2, 4, 8), (1, 2), (1, 2, 4), (2, 4, 8)):
    if kg * pw > 8 or tn * 14 > 32 * pw:
        continue
    specs.append(f"ver=2,tk=8,tw=14,kg={kg},pw={pw},tn={tn},th=14,bc={bc}")
for spec in specs:
    try:
        plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
    except conv.ConvError as e:
        print(json.dumps({"spec": spec, "error": str(e)[:90]}), flush=True)
        continue
    o, ws = plan.new_output(), plan.new_workspace()
    us = timeit(plan, i, k, o, ws)
    got = o[:2].cpu().numpy().astype(np.float64)
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    d = plan.describe()
    print(json.dumps({"spec": spec, "tile": d["tile"], "us": round(us, 1), "tflops": round(sh.flops / us / 1e6, 2),
                      "model_us": round(d["model"]["model_us"], 1), "rel": rel}), flush=True)

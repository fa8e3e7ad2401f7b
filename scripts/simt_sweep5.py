"""SIMT batched-layer sweep over the row-mode family (TW = W, TK = 4): kg, tn,
th, bc -- bench protocol timing + relL2 of two images vs the oracle."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs  # noqa: E402
from scripts.simt_sweep4 import timeit  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "batched"
sh = CONFIGS[name]
xi, wi = make_inputs(sh, seed=0)
i, k = xi.cuda(), wi.cuda()
ref = oracle.conv_eq1(xi.numpy()[:2], wi.numpy())
specs = [None]
for kg, tn, th, bc in itertools.product((4, 8, 16), (1, 2, 4, 16), (14, 2), (2, 4, 8, 16)):
    slots = tn * th
    pw = (slots + 31) // 32
    if 32 * kg * pw > 512:
        continue
    specs.append(f"ver=2,tk=4,tw={sh.W},kg={kg},pw={pw},tn={tn},th={th},bc={bc}")
for spec in specs:
    try:
        plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
    except conv.ConvError as e:
        continue
    o, ws = plan.new_output(), plan.new_workspace()
    us = timeit(plan, i, k, o, ws)
    got = o[:2].cpu().numpy().astype(np.float64)
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    d = plan.describe()
    print(json.dumps({"spec": spec, "tile": d["tile"], "us": round(us, 1), "tflops": round(sh.flops / us / 1e6, 2),
                      "model_us": round(d["model"]["model_us"], 1), "rel": rel}), flush=True)

"""SIMT v2 TMA layout A/B (r02): one JSON line per (config, N, tile spec) with
the bench-protocol time, TFLOP/s, the modeled time and the relL2 of the first
two images against the oracle.  Run once as is and once with
CONV_SIMT_NO_TMA=1 (the per-thread cp.async layout) to compare.

Usage: python scripts/simt_sweep7.py [config] [N,N,...] [spec;spec;...]"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs  # noqa: E402
from scripts.simt_sweep4 import timeit  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "batched"
base = CONFIGS[name]
ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 and sys.argv[2] else [base.N]
specs = sys.argv[3].split(";") if len(sys.argv) > 3 else [""]
tma = "off" if os.environ.get("CONV_SIMT_NO_TMA") else "on"
for n in ns:
    sh = dataclasses.replace(base, N=n)
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    ref = oracle.conv_eq1(xi.numpy()[:2], wi.numpy())
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec or None)
        except conv.ConvError as e:
            print(json.dumps({"N": n, "spec": spec, "error": str(e)[:90]}), flush=True)
            continue
        o, ws = plan.new_output(), plan.new_workspace()
        us = timeit(plan, i, k, o, ws)
        got = o[:2].cpu().numpy().astype(np.float64)
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        d = plan.describe()
        print(json.dumps({"config": name, "N": n, "tma": tma, "spec": spec, "tile": d["tile"], "us": round(us, 1),
                          "tflops": round(sh.flops / us / 1e6, 2), "model_us": round(d["model"]["model_us"], 1),
                          "rel": rel}), flush=True)

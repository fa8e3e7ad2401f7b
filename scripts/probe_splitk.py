"""Split-K study script: per-kernel times (CUDA events between the kernels,
L2 flushed before each step) of a few small-M Table-1 layers for forced
split counts.  Usage: python scripts/probe_splitk.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import TABLE1, make_inputs  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device=dev)
for name in ("R6", "M7", "M9", "R12"):
    sh = TABLE1[name]
    inp, ker = make_inputs(sh, seed=0)
    i, k = inp.to(dev), ker.to(dev)
    for sp in (1, 2, 4, 6, 8):
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="bf16", tile=f"splits={sp}", **sh.plan_kwargs())
        except conv.ConvError:
            continue
        out, ws = plan.new_output(dev), plan.new_workspace(dev)
        nk = plan.num_kernels
        for _ in range(3):
            plan.run(i, k, out, ws)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)] for _ in range(20)]
        tot = []
        for e in ev:
            flush.zero_()
            plan.run_events(i, k, out, ws, e)
        torch.cuda.synchronize()
        kern = [float(np.median([e[j].elapsed_time(e[j + 1]) for e in ev])) * 1e3 for j in range(nk)]
        print(json.dumps({"layer": name, "splits": sp, "tile": plan.describe()["tile"],
                          "kernels_us": [round(x, 2) for x in kern]}),
              flush=True)

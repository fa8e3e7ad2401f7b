"""r02b: FP32 SIMT time of Table-1 layers with the AUTO tile and with forced
wider register tiles (TK = 8, TW = 8), which need fewer shared-memory
wavefronts per FMA.  Usage: python scripts/probe_simt_tiles_t1.py LAYER,... SPEC;SPEC"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import TABLE1, make_inputs  # noqa: E402
from scripts.simt_sweep4 import timeit  # noqa: E402

layers = sys.argv[1].split(",")
specs = [""] + (sys.argv[2].split(";") if len(sys.argv) > 2 else [])
for name in layers:
    sh = TABLE1[name]
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec or None, **sh.plan_kwargs())
        except conv.ConvError as e:
            print(json.dumps({"layer": name, "spec": spec, "error": str(e)[:80]}), flush=True)
            continue
        o, ws = plan.new_output(), plan.new_workspace()
        us = timeit(plan, i, k, o, ws)
        d = plan.describe()
        print(json.dumps({"layer": name, "spec": spec, "tile": d["tile"], "us": round(us, 1),
                          "model_us": round(d["model"]["model_us"], 1)}), flush=True)

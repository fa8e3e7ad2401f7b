python - <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
from scripts.simt_sweep4 import timeit
sh = CONFIGS["det"]
xi, wi = make_inputs(sh, seed=0); i, k = xi.cuda(), wi.cuda()
specs = ["", "th=1", "th=2", "th=3", "th=4", "th=6", "th=8",
         "tw=8,th=2", "tw=8,th=4", "tw=8,th=6", "tw=8,kg=4,th=4", "tw=8,kg=2,th=8", "tw=4,kg=4,th=4", "tw=4,kg=2,th=6",
         "tk=8,tw=4,th=4", "tk=8,tw=8,th=4", "tk=8,tw=8,kg=2,th=6", "tw=8,th=4,splits=2", "tw=4,th=4,splits=2"]
for spec in specs:
    try:
        plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec or None)
    except conv.ConvError as e:
        print(json.dumps({"spec": spec, "error": str(e)[:60]})); continue
    o, ws = plan.new_output(), plan.new_workspace()
    us = timeit(plan, i, k, o, ws)
    d = plan.describe()
    print(json.dumps({"spec": spec, "tile": d["tile"], "us": round(us, 1), "model_us": round(d["model"]["model_us"], 1)}), flush=True)
PY

"""SIMT tile study under the bench protocol (CUDA-graph replay, L2 flushed before every step):
every v2 candidate tile (tk, tw, kg, tn, bc) and v1 candidate (tk, tw, kg, bc) of a layer, modeled vs measured (selector
calibration for the latency-bound small layers).  Product code only."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, make_inputs
from scripts.selector_study import time_plan, spearman
torch.cuda.set_device(0)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(max(2 * l2, 256 << 20) // 4, device="cuda"); flush_rd = torch.ones_like(flush); fo = torch.empty((), device="cuda")
for name in sys.argv[1].split(","):
    sh = CONFIGS[name] if name in CONFIGS else TABLE1[name]
    inp, ker = make_inputs(sh); i, k = inp.cuda(), ker.cuda()
    auto = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", **sh.plan_kwargs()).describe()["tile"]
    rows = []
    specs = [f"ver=2,tk={tk},tw={tw},kg={kg},tn={tn},bc={bc}"
             for tk, tw, kg, tn, bc in itertools.product((4, 8), (4, 8, sh.W), (1, 2, 4, 8), (1, 2, 4), (4, 8, 16))]
    # v1 (any R, S, stride): the selector fills th / pw / tn
    specs += [f"ver=1,tk={tk},tw={tw},kg={kg},bc={bc}"
              for tk, tw, kg, bc in itertools.product((4, 8), (1, 2, 4), (1, 2, 4, 8), (4, 8, 16, 32))]
    for spec in specs:
        try:
            p = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec, **sh.plan_kwargs())
        except conv.ConvError:
            continue
        d = p.describe()
        if any(r["tile"] == d["tile"] for r in rows):
            continue
        rows.append({"tile": d["tile"], "model_us": d["model"]["model_us"], "us": time_plan(p, i, k, flush, flush_rd, fo)})
    m = np.array([r["model_us"] for r in rows]); t = np.array([r["us"] for r in rows])
    a = [r for r in rows if r["tile"] == auto]
    if not a:   # the AUTO tile (e.g. split-C) is not among the forced, unsplit tiles: time it
        ap = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", **sh.plan_kwargs())
        a = [{"tile": auto, "model_us": ap.describe()["model"]["model_us"], "us": time_plan(ap, i, k, flush, flush_rd, fo)}]
    print(json.dumps({"layer": name, "n": len(rows), "best_us": round(float(t.min()), 1), "best": rows[int(t.argmin())]["tile"],
                      "auto_us": round(a[0]["us"], 1) if a else None, "auto": auto, "rho": round(spearman(m, t), 2),
                      "rows": [{"tile": r["tile"], "model": round(r["model_us"], 1), "us": round(r["us"], 1)} for r in rows]}), flush=True)

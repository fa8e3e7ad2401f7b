"""Offline check of the SIMT model against a measured tile study
(scripts/simt_study.py output): for every measured tile, the current
library's modeled time; per layer the measured time of the model's pick
among the measured tiles, its loss vs the measured best, and Spearman rho.
CPU only.  Usage: python scripts/simt_model_eval.py study.jsonl"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1  # noqa: E402

DEV = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
tot_pick = tot_best = 0.0
for line in open(sys.argv[1]):
    j = json.loads(line)
    sh = CONFIGS[j["layer"]] if j["layer"] in CONFIGS else TABLE1[j["layer"]]
    rows = []
    for r in j["rows"]:
        t = r["tile"]
        spec = ",".join(f"{k}={t[k]}" for k in ("ver", "tk", "tw", "kg", "pw", "tn", "th", "bc"))
        try:
            d = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec, offline_device=DEV,
                              **sh.plan_kwargs()).describe()
        except conv.ConvError:
            continue
        rows.append((d["model"]["model_us"], r["us"], t))
    if any(x[2]["ver"] == 2 for x in rows):      # the selector considers v1 only where v2 cannot run
        rows = [x for x in rows if x[2]["ver"] == 2]
    m = np.array([x[0] for x in rows])
    u = np.array([x[1] for x in rows])
    pick = u[int(m.argmin())]
    best = u.min()
    rho = np.corrcoef(np.argsort(np.argsort(m)), np.argsort(np.argsort(u)))[0, 1]
    auto = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", offline_device=DEV, **sh.plan_kwargs()).describe()["tile"]
    auto_meas = [x[1] for x in rows if x[2] == auto]
    tot_pick += pick
    tot_best += best
    print(f"{j['layer']:8s} pick {pick:8.1f}  best {best:8.1f}  loss {pick / best - 1:6.2%}  rho {rho:5.2f}  "
          f"auto measured {auto_meas[0] if auto_meas else 'n/a'}")
print(f"total pick {tot_pick:.1f} best {tot_best:.1f} loss {tot_pick / tot_best - 1:.2%}")

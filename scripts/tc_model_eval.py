"""Offline check of the tensor-path model against a measured tile study
(scripts/selector_study.py output): for every measured (bn, cg, kbs, fuse)
family the current library's modeled time (offline plan, same forced keys),
per layer the measured time of the model's pick, its loss vs the measured
best, and the mean loss.  CPU only.  Usage: tc_model_eval.py study.jsonl"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1  # noqa: E402

DEV = dict(sms=148, smem_optin=232448, l2_bytes=132120576)
losses = []
for line in open(sys.argv[1]):
    j = json.loads(line)
    sh = CONFIGS[j["layer"]] if j["layer"] in CONFIGS else TABLE1[j["layer"]]
    rows = []
    for r in j["rows"]:
        try:
            d = conv.ConvPlan(*sh.as_tuple(), path=j["path"], tile=r["spec"], offline_device=DEV,
                              **sh.plan_kwargs()).describe()
        except conv.ConvError:
            continue
        rows.append((d["model"]["model_us"], r["measured_us"]))
    m = np.array([x[0] for x in rows])
    u = np.array([x[1] for x in rows])
    pick, best = u[int(m.argmin())], u.min()
    losses.append(pick / best - 1)
    print(f"{j['layer']:8s} pick {pick:8.2f} best {best:8.2f} loss {pick / best - 1:6.2%}")
print(f"mean loss {np.mean(losses):.2%}  max {max(losses):.2%}")

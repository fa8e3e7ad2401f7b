"""Selector validation study, the B200 analog of
the paper's Sec. 9 evaluation (Fig. 5): for each layer,
every feasible tensor-path tile (bn x cg x kbs x fuse, stages = the most that
fit) is planned -- the model's predicted time comes from conv_plan_describe --
and measured with the bench protocol (CUDA-graph replay of conv_run, L2
flushed before every step outside the event pair).  Reported per layer:

* top-k loss (k = 1, 2, 5): best measured time among the k configurations
  the model ranks first, over the best measured time of all, minus 1
  (PAPER.md:483's "loss-of-performance");
* Spearman rank correlation between modeled and measured times;
* the selector's own pick (AUTO tile of the path) and its loss.

Product code only (no oracle): correctness of every forced tile is covered
by tests/test_parity.py.  Usage: python scripts/selector_study.py [bf16|tf32]
[layer,...] > profiles/.../selector_study.jsonl
"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, make_inputs  # noqa: E402

DEFAULT_LAYERS = ["r2", "pw", "det", "batched", "Y2", "Y8", "Y12", "Y23", "R4", "R8", "R12", "M3", "M7", "M9"]


def shape_of(name):
    return CONFIGS[name] if name in CONFIGS else TABLE1[name]


def time_plan(plan, d_in, d_ker, flush, flush_rd, flush_out, steps=15):
    out, ws = plan.new_output(), plan.new_workspace()
    stream = torch.cuda.current_stream()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        for _ in range(3):
            plan.run(d_in, d_ker, out, ws, stream=cap)
    cap.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        plan.run(d_in, d_ker, out, ws, stream=cap)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_out)
        a.record(stream)
        g.replay()
        b.record(stream)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def spearman(x, y):
    rx = np.argsort(np.argsort(x)).astype(float)
    ry = np.argsort(np.argsort(y)).astype(float)
    return float(np.corrcoef(rx, ry)[0, 1]) if len(x) > 2 else float("nan")


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    layers = sys.argv[2].split(",") if len(sys.argv) > 2 else DEFAULT_LAYERS
    torch.cuda.set_device(0)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, device="cuda")
    flush_rd = torch.ones_like(flush)
    flush_out = torch.empty((), device="cuda")
    for name in layers:
        sh = shape_of(name)
        inp, ker = make_inputs(sh, seed=0)
        d_in, d_ker = inp.cuda(), ker.cuda()
        auto = conv.ConvPlan(*sh.as_tuple(), path=path, **sh.plan_kwargs())
        auto_tile = auto.describe()["tile"]
        rows = []
        for bn, cg, kbs, fuse in itertools.product((32, 64, 128, 192, 256), (1, 2), (1, 2, 3, 4, 6, 7, 9), (0, 1)):
            spec = f"bn={bn},cg={cg},kbs={kbs},fuse={fuse}"
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
            except conv.ConvError:
                continue
            d = plan.describe()
            us = time_plan(plan, d_in, d_ker, flush, flush_rd, flush_out)
            t = d["tile"]
            rows.append({"spec": spec, "tile": t, "model_us": d["model"]["model_us"], "measured_us": us,
                         "auto": all(t[k] == auto_tile[k] for k in ("bn", "cg", "kbs", "fuse", "stages"))})
        model = np.array([r["model_us"] for r in rows])
        meas = np.array([r["measured_us"] for r in rows])
        best = meas.min()
        order = np.argsort(model)
        loss = {f"top{k}": float(meas[order[:k]].min() / best - 1.0) for k in (1, 2, 5)}
        auto_rows = [r for r in rows if r["auto"]]
        auto_us = auto_rows[0]["measured_us"] if auto_rows else time_plan(auto, d_in, d_ker, flush, flush_rd, flush_out)
        print(json.dumps({"layer": name, "path": path, "configs": len(rows), "best_us": round(float(best), 2),
                          "best_tile": rows[int(meas.argmin())]["spec"], "auto_tile": auto_tile,
                          "auto_us": round(auto_us, 2), "auto_loss": round(auto_us / best - 1.0, 4),
                          "loss": {k: round(v, 4) for k, v in loss.items()},
                          "spearman": round(spearman(model, meas), 3),
                          "rows": [{"spec": r["spec"], "model_us": round(r["model_us"], 2),
                                    "measured_us": round(r["measured_us"], 2)} for r in rows]}), flush=True)


if __name__ == "__main__":
    main()

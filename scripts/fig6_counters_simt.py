"""Model vs hardware counters for the FP32 SIMT path (the headline path's leg
of NEXT-3 / the paper's Fig. 6; the tensor
paths' leg is scripts/fig6_counters.py).

For each layer a set of forced SIMT tiles (register tile, k groups, channel
chunk, images per tile, flat row mode, split-C) is planned; the selector's
modeled volumes come from conv_plan_describe (DV_{L2->SMEM}: every CTA loads
its In halo tile and Ker slab once per channel chunk, Eq. 4's footprints;
DV_HBM: compulsory bytes + the packed Ker) and each plan runs ONCE under ncu:

  run:     ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,
               lts__t_sectors_op_read.sum,gpu__time_duration.sum --csv --page raw --log-file counters.csv
               python scripts/fig6_counters_simt.py run LAYER[,LAYER..] [STRIDE] > manifest.jsonl
  analyze: python scripts/fig6_counters_simt.py analyze manifest.jsonl counters.csv > fig6_simt.jsonl

Per layer: Spearman rank correlation over the tiles between the modeled
volume and the counter (L2 read sectors x 32 B of the convolution grids --
main + remainder), the median counter / model ratio, and the same between
the modeled time and the kernels' measured duration.
"""
import dataclasses
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.fig6_counters import launches, spearman  # noqa: E402


def shape_of(name):
    from paper_2101_09808_b200.inputs import CONFIGS, TABLE1
    if name.startswith("batched"):                      # batched64: the 64-image shard
        n = name[len("batched"):]
        return dataclasses.replace(CONFIGS["batched"], N=int(n)) if n else CONFIGS["batched"]
    return CONFIGS[name] if name in CONFIGS else TABLE1[name]


def run(layers, stride=1):
    import torch

    from paper_2101_09808_b200 import conv
    from paper_2101_09808_b200.inputs import make_inputs
    torch.cuda.set_device(0)
    for name in layers:
        sh = shape_of(name)
        inp, ker = make_inputs(sh, seed=0)
        d_in, d_ker = inp.cuda(), ker.cuda()
        seen = set()
        for flat, tk, tw, kg, bc, tn, sp in itertools.product((0, 1), (4, 8), (4, 8, 7, 14), (1, 2, 4, 8), (4, 8, 16),
                                                              (1, 2, 4), (1, 2)):
            if flat and tn != 1:
                continue
            spec = f"ver=2,flat={flat},tk={tk},tw={tw},kg={kg},bc={bc},splits={sp}" + ("" if flat else f",tn={tn}")
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec, **sh.plan_kwargs())
            except conv.ConvError:
                continue
            d = plan.describe()
            t = d["tile"]
            key = json.dumps(t, sort_keys=True)
            if key in seen:
                continue
            seen.add(key)
            if (len(seen) - 1) % stride:                 # every stride-th distinct tile
                continue
            out, ws = plan.new_output(), plan.new_workspace()
            torch.cuda.synchronize()
            plan.run(d_in, d_ker, out, ws)
            torch.cuda.synchronize()
            lv = d["model"]["levels"]
            print(json.dumps({"layer": name, "spec": spec, "tile": t,
                              "launches": 2 + (1 if t["rem"] > 0 else 0) + (1 if t["splits"] > 1 else 0),
                              "dv_l2_smem": lv["l2_smem"]["dv_bytes"], "dv_hbm": lv["hbm"]["dv_bytes"],
                              "model_us": d["model"]["model_us"]}), flush=True)


def analyze(manifest, counters):
    import numpy as np
    tiles = [json.loads(l) for l in open(manifest) if l.startswith("{")]
    ks = [k for k in launches(counters) if "conv_direct_simt" in k[0] or "pack_ker_simt" in k[0] or "reduce_splits" in k[0]]
    pos = 0
    for t in tiles:
        group = ks[pos:pos + t["launches"]]
        pos += t["launches"]
        conv_k = [g[1] for g in group if "conv_direct_simt" in g[0]]
        t["l2_read_bytes"] = 32.0 * sum(c.get("lts__t_sectors_srcunit_tex_op_read.sum", 0.0) for c in conv_k)
        t["l2_read_all_bytes"] = 32.0 * sum(c.get("lts__t_sectors_op_read.sum", 0.0) for c in conv_k)
        t["dram_bytes"] = sum(g[1].get("dram__bytes_read.sum", 0) + g[1].get("dram__bytes_write.sum", 0) for g in group)
        t["dram_read"] = sum(g[1].get("dram__bytes_read.sum", 0) for g in group)
        t["conv_ns"] = max(c.get("gpu__time_duration.sum", 0) for c in conv_k)   # the grids run side by side
        t["conv_all_ns"] = [c.get("gpu__time_duration.sum", 0) for c in conv_k]
        t["all_ns"] = [g[1].get("gpu__time_duration.sum", 0) for g in group]
    assert pos == len(ks), f"{pos} launches matched, {len(ks)} in the log"
    by = {}
    for t in tiles:
        by.setdefault(t["layer"], []).append(t)
    for layer, rows in by.items():
        m_l2 = np.array([r["dv_l2_smem"] for r in rows])
        c_l2 = np.array([r["l2_read_all_bytes"] for r in rows])
        m_hbm = np.array([r["dv_hbm"] for r in rows])
        c_hbm = np.array([r["dram_bytes"] for r in rows])
        m_t = np.array([r["model_us"] for r in rows])
        # ncu serialises the remainder grid and the main grid, which run side by side: count the longer
        c_t = np.array([(sum(r["all_ns"]) - (sum(r["conv_all_ns"]) - r["conv_ns"])) / 1e3 for r in rows])
        best_meas = int(np.argmin(c_t))
        best_model = int(np.argmin(m_t))
        print(json.dumps({
            "layer": layer, "tiles": len(rows),
            "l2_smem": {"spearman": round(spearman(m_l2, c_l2), 3),
                        "median_counter_over_model": round(float(np.median(c_l2 / m_l2)), 3),
                        "min_max_counter_over_model": [round(float((c_l2 / m_l2).min()), 3), round(float((c_l2 / m_l2).max()), 3)]},
            "hbm": {"model_bytes": float(m_hbm[0]), "dram_bytes_min_med_max": [float(c_hbm.min()), float(np.median(c_hbm)), float(c_hbm.max())],
                    "dram_read_med": float(np.median([r["dram_read"] for r in rows]))},
            "time": {"spearman": round(spearman(m_t, c_t), 3),
                     "model_pick": rows[best_model]["spec"], "model_pick_us_cold_serialised": round(float(c_t[best_model]), 1),
                     "best_measured": rows[best_meas]["spec"], "best_us": round(float(c_t[best_meas]), 1),
                     "top1_loss": round(float(c_t[best_model] / c_t[best_meas] - 1.0), 4)},
            "rows": [{"spec": r["spec"], "rem": r["tile"]["rem"], "dv_l2_smem": r["dv_l2_smem"], "l2_read": r["l2_read_all_bytes"],
                      "l2_read_tex": r["l2_read_bytes"], "dram": r["dram_bytes"], "model_us": r["model_us"],
                      "ns": r["all_ns"]} for r in rows],
        }), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2].split(","), int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    else:
        analyze(sys.argv[2], sys.argv[3])

"""Model vs hardware counters (the Fig. 6 leg of
the paper's Sec. 9: "the model-predicted data movement is compared with
hardware counter events").

For each layer, every feasible tensor-path tile (bn x cg x kbs x fuse) is
planned; the selector's per-level data volumes come from conv_plan_describe
(DV_{L2->SMEM}: the Sec. 3.2 model of the CTA tile's operand loads;
DV_HBM: compulsory bytes + layout transforms) and each plan runs ONCE, so
that an ncu launch list pairs every tile with its kernels' counters:

  run:     python scripts/fig6_counters.py run PATH LAYER[,LAYER..] > manifest.jsonl
           (under: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
            lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,gpu__time_duration.sum
            --csv --page raw --log-file counters.csv  python scripts/fig6_counters.py run ...)
  analyze: python scripts/fig6_counters.py analyze manifest.jsonl counters.csv > fig6.jsonl

ncu flushes the caches before every kernel (--cache-control all), the
cold-L2 protocol of the bench.  Per layer and level the report gives the
Spearman rank correlation between the model's volume and the counter over
the tiles (the paper's Fig. 6 statistic) and the median counter / model
ratio.  Measured: main kernel L2 -> SM reads (lts sectors read x 32 B) vs
DV_{L2->SMEM}; DRAM read + write bytes of both kernels vs DV_HBM.
"""
import csv
import io
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LAYERS = {"R9": (1, 256, 256, 14, 14, 3, 3), "Y5": (1, 64, 128, 136, 136, 1, 1)}


def shape_of(name):
    from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, Shape
    if name in LAYERS:
        return Shape(*LAYERS[name])
    return CONFIGS[name] if name in CONFIGS else TABLE1[name]


def run(path, layers):
    import torch

    from paper_2101_09808_b200 import conv
    from paper_2101_09808_b200.inputs import make_inputs
    torch.cuda.set_device(0)
    for name in layers:
        sh = shape_of(name)
        inp, ker = make_inputs(sh, seed=0)
        d_in, d_ker = inp.cuda(), ker.cuda()
        for bn, cg, kbs, fuse in itertools.product((32, 64, 128, 192, 256), (1, 2), (1, 2, 3, 4, 6, 9), (0, 1)):
            spec = f"bn={bn},cg={cg},kbs={kbs},fuse={fuse},splits=1"
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
            except conv.ConvError:
                continue
            d = plan.describe()
            out, ws = plan.new_output(), plan.new_workspace()
            torch.cuda.synchronize()
            plan.run(d_in, d_ker, out, ws)
            torch.cuda.synchronize()
            lv = d["model"]["levels"]
            print(json.dumps({"layer": name, "path": path, "spec": spec, "tile": d["tile"], "kernels": d["kernels"],
                              "dv_l2_smem": lv["l2_smem"]["dv_bytes"], "dv_hbm": lv["hbm"]["dv_bytes"],
                              "model_us": d["model"]["model_us"]}), flush=True)


def spearman(x, y):
    import numpy as np
    rx = np.argsort(np.argsort(x)).astype(float)
    ry = np.argsort(np.argsort(y)).astype(float)
    return float(np.corrcoef(rx, ry)[0, 1]) if len(x) > 2 else float("nan")


def launches(csv_path):
    """Kernel rows of an ncu --csv --page raw log: [(name, {metric: value})]."""
    text = open(csv_path).read()
    i0 = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[i0:])))
    hdr = rows[0]
    out = []
    for r in rows[2:]:                          # row 1 holds the units
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        vals = {}
        for k, v in d.items():
            if "__" in k:
                try:
                    vals[k] = float(v.replace(",", ""))
                except ValueError:
                    pass
        out.append((d.get("Kernel Name", ""), vals))
    return out


def analyze(manifest, counters):
    import numpy as np
    tiles = [json.loads(l) for l in open(manifest) if l.startswith("{")]
    ks = [k for k in launches(counters) if "conv_igemm" in k[0] or "repack" in k[0] or "expand" in k[0]]
    pos = 0
    for t in tiles:
        n = t["kernels"]
        group = ks[pos:pos + n]
        pos += n
        main = group[-1][1]
        t["l2_read_bytes"] = 32.0 * main.get("lts__t_sectors_srcunit_tex_op_read.sum", main.get("lts__t_sectors_op_read.sum", 0.0))
        t["l2_read_all_bytes"] = 32.0 * main.get("lts__t_sectors_op_read.sum", 0.0)
        t["dram_bytes"] = sum(g[1].get("dram__bytes_read.sum", 0) + g[1].get("dram__bytes_write.sum", 0) for g in group)
        t["dram_read"] = sum(g[1].get("dram__bytes_read.sum", 0) for g in group)
        t["dram_write"] = sum(g[1].get("dram__bytes_write.sum", 0) for g in group)
        t["kernel_ns"] = [g[1].get("gpu__time_duration.sum", 0) for g in group]
    assert pos == len(ks), f"{pos} launches matched, {len(ks)} in the log"
    by = {}
    for t in tiles:
        by.setdefault((t["layer"], t["path"]), []).append(t)
    for (layer, path), rows in by.items():
        m_l2 = np.array([r["dv_l2_smem"] for r in rows])
        c_l2 = np.array([r["l2_read_bytes"] for r in rows])
        m_hbm = np.array([r["dv_hbm"] for r in rows])
        c_hbm = np.array([r["dram_bytes"] for r in rows])
        sh = shape_of(layer)
        comp_read = 4.0 * (sh.N * sh.C * sh.Hin * sh.Win + sh.K * sh.C * sh.R * sh.S)
        comp_write = 4.0 * sh.N * sh.K * sh.H * sh.W
        classes = {}
        for fz in (0, 1):
            rr = [r for r in rows if r["tile"]["fuse"] == fz]
            if rr:
                d = np.array([r["dram_bytes"] for r in rr])
                classes[f"fuse{fz}"] = {
                    "tiles": len(rr), "model_bytes": rr[0]["dv_hbm"],
                    "dram_bytes_min_med_max": [float(d.min()), float(np.median(d)), float(d.max())],
                    "dram_read_med": float(np.median([r["dram_read"] for r in rr])),
                    "dram_write_med": float(np.median([r["dram_write"] for r in rr]))}
        print(json.dumps({
            "layer": layer, "path": path, "tiles": len(rows),
            "compulsory_read_bytes": comp_read, "compulsory_write_bytes": comp_write, "hbm_classes": classes,
            "l2_smem": {"spearman": round(spearman(m_l2, c_l2), 3),
                        "median_counter_over_model": round(float(np.median(c_l2 / m_l2)), 3)},
            "hbm": {"spearman": round(spearman(m_hbm, c_hbm), 3),
                    "median_counter_over_model": round(float(np.median(c_hbm / m_hbm)), 3)},
            "rows": [{"spec": r["spec"], "dv_l2_smem": r["dv_l2_smem"], "l2_read": r["l2_read_bytes"],
                      "dv_hbm": r["dv_hbm"], "dram": r["dram_bytes"], "kernel_ns": r["kernel_ns"]} for r in rows],
        }), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3].split(","))
    else:
        analyze(sys.argv[2], sys.argv[3])

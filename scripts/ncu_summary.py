"""Summarise ncu captures (launch lists + --set full reports) into profiles/."""
import csv, io, json, subprocess, sys, os

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpc__cycles_elapsed.max", "sm__cycles_active.avg", "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k:
                    d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res

def launches(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    out = [(r[ki], float(r[vi])) for r in rows[i0 + 1:] if len(r) > vi]
    return out

if __name__ == "__main__":
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    lists = [a for a in sys.argv[2:] if a.endswith(".csv")]
    summary = {"tag": tag, "reports": {}, "launch_lists": {}}
    for rep in reps:
        summary["reports"][os.path.basename(rep)] = raw(rep)
    for l in lists:
        ls = launches(l)
        agg = {}
        for k, v in ls:
            name = k.split("(")[0].replace("void ", "")
            agg.setdefault(name, []).append(v)
        summary["launch_lists"][os.path.basename(l)] = {
            n: {"launches": len(v), "mean_ns": sum(v) / len(v), "min_ns": min(v), "max_ns": max(v)} for n, v in agg.items()}
    print(json.dumps(summary, indent=1))

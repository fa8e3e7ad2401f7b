"""Single-thread and all-core oracle times for the BASELINE configs (BASELINE.md
Sec. 3: the CPU baseline beside the GPU results; one image of the batched
layer).  Test infrastructure: the oracle only.  Usage:
python scripts/oracle_single_thread.py > profiles/.../oracle_times.jsonl"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, Shape, make_inputs  # noqa: E402

allc = oracle.num_threads(oracle.host_threads())
for name, sh in CONFIGS.items():
    if name == "batched":
        sh = Shape(1, sh.K, sh.C, sh.H, sh.W, sh.R, sh.S)
    inp, ker = make_inputs(sh, seed=0)
    x, w = inp.numpy(), ker.numpy()
    row = {"config": name + (" (1 image)" if name == "batched" else ""), "gflop": sh.flops / 1e9}
    for th in (1, allc):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            oracle.conv_eq1(x, w, nthreads=th)
            ts.append(time.perf_counter() - t0)
        t = min(ts)                                  # best of 3
        row[f"threads_{th}"] = {"s": round(t, 5), "gflops": round(sh.flops / t / 1e9, 3)}
    row["cpu"] = open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip()
    print(json.dumps(row), flush=True)

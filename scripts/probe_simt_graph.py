"""Study script: one SIMT layer timed three ways under the bench's L2 flush --
CUDA-graph replay of conv_run, plain stream launches of conv_run, and
conv_run_events (events between the kernels).  Usage: probe_simt_graph.py LAYER..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import TABLE1, make_inputs  # noqa: E402

flush = torch.empty(256 << 20 >> 2, device="cuda")
flush_rd = torch.ones_like(flush)
fo = torch.empty((), device="cuda")
st = torch.cuda.current_stream()


def timed(fn, n=10):
    ts = []
    for _ in range(n):
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=fo)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for name in sys.argv[1:]:
    sh = TABLE1[name]
    inp, ker = make_inputs(sh, seed=0)
    i, k = inp.cuda(), ker.cuda()
    plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", **sh.plan_kwargs())
    out, ws = plan.new_output(), plan.new_workspace()
    for _ in range(3):
        plan.run(i, k, out, ws)
    cap = torch.cuda.Stream()
    cap.wait_stream(st)
    with torch.cuda.stream(cap):
        plan.run(i, k, out, ws, stream=cap)
    cap.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        plan.run(i, k, out, ws, stream=cap)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_graph = timed(g.replay)
    t_plain = timed(lambda: plan.run(i, k, out, ws))

    def run_ev():
        plan.run_events(i, k, out, ws, ev)
    t_ev = timed(run_ev)
    print(name, plan.describe()["tile"], f"graph {t_graph:.1f} plain {t_plain:.1f} events {t_ev:.1f} "
          f"(kernels {ev[0].elapsed_time(ev[1]) * 1e3:.1f} + {ev[1].elapsed_time(ev[2]) * 1e3:.1f}) us", flush=True)

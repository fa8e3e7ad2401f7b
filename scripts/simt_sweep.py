"""Parity + timing of SIMT tiles (selector choice and forced variants)."""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs

def timeit(plan, i, k, o, ws, n=10):
    for _ in range(2): plan.run(i, k, o, ws)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_kernels + 1)]
    ts = []
    for _ in range(n):
        plan.run_events(i, k, o, ws, ev); torch.cuda.synchronize()
        ts.append(ev[-2].elapsed_time(ev[-1]))
    return float(np.median(ts)) * 1e3

for name in sys.argv[1:]:
    sh = CONFIGS[name]
    xi, wi = make_inputs(sh, seed=1, kind="int")
    n_check = min(sh.N, 2)
    ref = oracle.conv_eq1(xi.numpy()[:n_check], wi.numpy())
    i, k = xi.cuda(), wi.cuda()
    specs = [None, "ver=1"]
    for tk, tw, kg in itertools.product((4, 8), (4, 8), (1, 2, 4)):
        specs.append(f"ver=2,tk={tk},tw={tw},kg={kg}")
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        except conv.ConvError as e:
            print(f"{name} {spec}: infeasible ({e})"); continue
        o = plan.new_output(); ws = plan.new_workspace()
        plan.run(i, k, o, ws); torch.cuda.synchronize()
        ok = np.array_equal(o.cpu().numpy()[:n_check].astype(np.float64), ref)
        us = timeit(plan, i, k, o, ws)
        d = plan.describe()
        print(f"{name:8s} {str(spec):28s} exact={ok} main={us:9.2f}us  {sh.flops/us/1e6:6.2f} TF/s  model={d['model']['model_us']:8.2f}  tile={d['tile']}", flush=True)

"""Wider SIMT v2 sweep: measured vs modeled time (selector calibration)."""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
from scripts.simt_sweep import timeit
for name in sys.argv[1:]:
    sh = CONFIGS[name]
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    res = []
    specs = [None] + [f"ver=2,tk={tk},tw={tw},kg={kg},tn={tn},bc={bc}" for tk, tw, kg, tn, bc in
                      itertools.product((4, 8), (4, 8), (1, 2, 4, 8), (1, 2, 4), (4, 8, 16))]
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        except conv.ConvError:
            continue
        o = plan.new_output(); ws = plan.new_workspace()
        us = timeit(plan, i, k, o, ws, n=5)
        d = plan.describe()
        res.append((us, d['model']['model_us'], str(spec), d['tile']))
    res.sort(key=lambda x: x[0])
    sel = [r for r in res if r[2] == 'None'][0]
    print(f"== {name}: selector pick {sel[0]:.1f}us (model {sel[1]:.1f}) {sel[3]}")
    for us, m, spec, tile in res[:12]:
        print(f"  {us:9.1f}us  {sh.flops/us/1e6:6.2f} TF/s  model={m:8.1f}  {tile}")
    ms = np.array([r[1] for r in res]); me = np.array([r[0] for r in res])
    print(f"  rank corr (model vs measured): {np.corrcoef(np.argsort(np.argsort(ms)), np.argsort(np.argsort(me)))[0,1]:.2f}  n={len(res)}")

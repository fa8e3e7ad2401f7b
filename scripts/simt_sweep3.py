"""SIMT row-mode sweep (TW = W): measured vs modeled time, batched-style layers."""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
from scripts.simt_sweep import timeit
import oracle
for name in sys.argv[1:]:
    sh = CONFIGS[name]
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    res = []
    specs = [None, "ver=2,tk=8,tw=4,kg=4,pw=1,tn=4,bc=8"]
    specs += [f"ver=2,tk=4,tw={sh.W},kg={kg},pw={pw},tn={tn},bc={bc}" for kg, pw, tn, bc in
              itertools.product((2, 4, 8), (1, 2), (4, 8, 16, 32), (4, 8, 16))]
    ref = None
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        except conv.ConvError:
            continue
        o = plan.new_output(); ws = plan.new_workspace()
        us = timeit(plan, i, k, o, ws, n=5)
        if ref is None:
            ref = oracle.conv_eq1(xi.numpy()[:2], wi.numpy())
        got = o[:2].cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        d = plan.describe()
        res.append((us, d['model']['model_us'], str(spec), d['tile'], rel))
    res.sort(key=lambda x: x[0])
    sel = [r for r in res if r[2] == 'None'][0]
    print(f"== {name}: selector pick {sel[0]:.1f}us (model {sel[1]:.1f}) {sel[3]}")
    for us, m, spec, tile, rel in res[:16]:
        print(f"  {us:9.1f}us  {sh.flops/us/1e6:6.2f} TF/s  model={m:8.1f} rel={rel:.1e} {tile}")
    print("  worst rel", max(r[4] for r in res))

import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import TABLE1, make_inputs

for name in sys.argv[1].split(","):
    sh = TABLE1[name]
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    for path in ("bf16", "tf32"):
        for spec in (None, "fuse=0", "fuse=1", "fuse=0,cg=1", "fuse=0,cg=2", "fuse=0,bn=64", "fuse=0,bn=128,cg=1"):
            try:
                plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=spec, **sh.plan_kwargs())
            except conv.ConvError as e:
                continue
            o = plan.new_output(); ws = plan.new_workspace()
            for _ in range(3): plan.run(i, k, o, ws)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_kernels + 1)]
            ts = []
            for _ in range(10):
                plan.run_events(i, k, o, ws, ev); torch.cuda.synchronize()
                ts.append([ev[j].elapsed_time(ev[j + 1]) * 1e3 for j in range(plan.num_kernels)])
            t = np.median(np.array(ts), axis=0)
            d = plan.describe()
            print(name, path, spec, [round(x, 1) for x in t], 'model', round(d['model']['model_us'], 1), d['tile'])

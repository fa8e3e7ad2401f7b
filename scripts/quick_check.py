"""Quick per-path parity + timing check on one config (one process per call so
that a faulting kernel cannot poison the others)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs

path, name = sys.argv[1], sys.argv[2]
tile = sys.argv[3] if len(sys.argv) > 3 else None
sh = CONFIGS[name]
plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile)
print(name, path, plan.describe()["tile"], flush=True)
for kind in ("int", "real"):
    inp, ker = make_inputs(sh, seed=1 if kind == "int" else 0, kind=kind)
    x = inp[:2].contiguous() if sh.N > 2 else inp
    out = plan.run(inp.cuda(), ker.cuda())
    torch.cuda.synchronize()
    got = out.cpu().numpy()[: x.shape[0]].astype(np.float64)
    ref = oracle.conv_eq1(x.numpy(), ker.numpy())
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(f"  {kind}: relL2={rel:.3e} exact={np.array_equal(got, ref)} maxabs={np.abs(got-ref).max():.3e}", flush=True)
    if kind == "int" and not np.array_equal(got, ref):
        bad = np.argwhere(got != ref)
        print("  first mismatches:", bad[:8].tolist(), got[tuple(bad[0])], ref[tuple(bad[0])])
i, k = inp.cuda(), ker.cuda()
o = plan.new_output(); ws = plan.new_workspace()
for _ in range(3): plan.run(i, k, o, ws)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_kernels + 1)]
ts = []
for _ in range(20):
    plan.run_events(i, k, o, ws, ev)
    torch.cuda.synchronize()
    ts.append([ev[j].elapsed_time(ev[j + 1]) * 1e3 for j in range(plan.num_kernels)])
ts = np.median(np.array(ts), axis=0)
main = ts[-1]
print(f"  kernel us: {np.round(ts, 2).tolist()}  main TFLOP/s={sh.flops / main / 1e6:.1f}  total TFLOP/s={sh.flops / ts.sum() / 1e6:.1f}")

"""Run the tensor kernel once with CONV_TRACE and summarise the per-CTA timeline.
Needs a trace build of the library: CONV_BUILD_TRACE=1 python -c "import
paper_2101_09808_b200.build as b; b.build(force=True)" (rebuild normally after)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path, cfg, tile = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "")
out = f"/tmp/trace_{path}_{cfg}_{tile.replace(',', '_').replace('=', '')}.bin"
env = dict(os.environ, CONV_TRACE=out)
code = f"""
import torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, make_inputs
sh = CONFIGS['{cfg}'] if '{cfg}' in CONFIGS else TABLE1['{cfg}']
p = conv.ConvPlan(*sh.as_tuple(), path='{path}', tile='{tile}' or None, **sh.plan_kwargs())
i, k = make_inputs(sh)
i, k = i.cuda(), k.cuda(); o = p.new_output(); ws = p.new_workspace()
for _ in range(3): p.run(i, k, o, ws)
torch.cuda.synchronize()
print(p.describe()['tile'])
"""
from paper_2101_09808_b200 import conv as _conv  # noqa: E402
if "+trace" not in _conv.load_library().conv_version().decode():
    raise SystemExit("not a trace build: CONV_BUILD_TRACE=1 python -c 'import paper_2101_09808_b200.build as b; "
                     "b.build(force=True)'")
subprocess.run([sys.executable, "-c", code], env=env, check=True)
t = np.fromfile(out, dtype=np.uint64).reshape(-1, 64).astype(np.int64)
t2all = t[512:]
t = t[:512]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print(f"CTAs traced: {len(t)}")
ntiles = [(t[c, 1:33].reshape(8, 4)[:, 0] > 0).sum() for c in range(len(t))]
print("tiles per CTA:", np.bincount(ntiles))
for ti in range(max(ntiles)):
    beg = t[:, 1 + 4 * ti] - t0; end = t[:, 3 + 4 * ti] - t0; wc = t[:, 2 + 4 * ti]
    ok = t[:, 1 + 4 * ti] > 0
    es, ee = t[:, 40 + 2 * ti] - t0, t[:, 41 + 2 * ti] - t0
    print(f"tile {ti}: mma begin {np.median(beg[ok])/1e3:7.2f}us  end {np.median(end[ok])/1e3:7.2f}us "
          f"(dur med {np.median((end-beg)[ok])/1e3:6.2f}us)  full-wait {np.median(wc[ok])/1e3:7.1f}kcyc  "
          f"epi {np.median(es[ok])/1e3:7.2f}->{np.median(ee[ok])/1e3:7.2f}us")
ends_ns = np.stack([t[:, 3 + 4 * i] for i in range(max(ntiles))], 1)
ends_clk = np.stack([t[:, 4 + 4 * i] for i in range(max(ntiles))], 1)
ok = (ends_ns[:, 0] > 0) & (ends_ns[:, -1] > 0)
mhz = (ends_clk[ok, -1] - ends_clk[ok, 0]) / (ends_ns[ok, -1] - ends_ns[ok, 0]) * 1e3
print(f"effective SM clock between first and last tile end: median {np.median(mhz):.0f} MHz (min {mhz.min():.0f}, max {mhz.max():.0f})")
print(f"producer empty-wait med {np.median(t[:,60])/1e3:.1f}kcyc, producer end med {np.median(t[:,61]-t0)/1e3:.2f}us")
n = max(ntiles)
last = np.max(t[:, 41 + 2 * (n - 1)] - t0)
print(f"last epilogue end {last/1e3:.2f}us; first start spread {(t[:,0].max()-t0)/1e3:.2f}us")
# fused transform (all CTAs, both ranks of a pair): slots 33-39, 56-58
a = np.fromfile(out, dtype=np.uint64).reshape(-1, 64).astype(np.int64)[:512]
f = a[a[:, 58] > 0]
f2 = t2all[:len(a)][a[:, 58] > 0]
if len(f):
    print(f"transform CTAs {len(f)}: chunks/CTA med {np.median(f[:,33]):.0f} (min {f[:,33].min()}, max {f[:,33].max()})")
    print(f"  start spread {(f[:,58].max()-f[:,58].min())/1e3:.2f}us, end med {np.median(f[:,38]-t0)/1e3:.2f}us max {np.max(f[:,38]-t0)/1e3:.2f}us")
    for k, name in ((34, "storer: wait converted"), (35, "storer: wait_read"), (36, "storer: bulk_wait lag"), (37, "storer: wait decoded")):
        print(f"  {name:30s} med {np.median(f[:,k])/1e3:8.1f} kcyc  max {f[:,k].max()/1e3:8.1f} kcyc")
    f2 = t2all[:len(a)][a[:, 58] > 0]
    for k, name in ((3, "decode 0,1 done"), (4, "first load issued"), (0, "chunk 0 converted"), (1, "first done report"), (2, "first publish")):
        print(f"  {name:26s} med {np.median(f2[:,k]-t0)/1e3:8.2f} us  max {np.max(f2[:,k]-t0)/1e3:8.2f} us")
    g = a[a[:, 56] > 0]
    print(f"  watcher sleep med {np.median(g[:,39])/1e3:.1f} kcyc, first unit ready med {np.median(g[:,56]-t0)/1e3:.2f}us")
    print(f"  producer ready-wait med {np.median(g[:,57])/1e3:.1f} kcyc max {g[:,57].max()/1e3:.1f}")

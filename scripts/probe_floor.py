"""Floor of the bench protocol for tiny steps: a CUDA graph of 1 / 2 trivial kernels timed like
bench.py (L2 flushed before every step outside the event pair, CUDA events around the replay),
next to the library's smallest layers (tiny / r2) on each path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
torch.cuda.set_device(0)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(max(2 * l2, 256 << 20) // 4, device="cuda"); flush_rd = torch.ones_like(flush); fo = torch.empty((), device="cuda")
def timed(g, steps=50):
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.zero_(); torch.sum(flush_rd, dim=0, out=fo)
        a.record(st); g.replay(); b.record(st)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
x = torch.zeros(1024, device="cuda")
for nk in (1, 2):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1)
    s.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(nk): x.add_(1)
    print(f"graph of {nk} trivial kernel(s): {timed(g):.2f} us")
for name in ("tiny", "r2"):
    sh = CONFIGS[name]
    inp, ker = make_inputs(sh); i, k = inp.cuda(), ker.cuda()
    for path in ("bf16", "tf32", "fp32_simt"):
        p = conv.ConvPlan(*sh.as_tuple(), path=path); o = p.new_output(); ws = p.new_workspace()
        s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            p.run(i, k, o, ws, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            p.run(i, k, o, ws, stream=s)
        print(f"{name} {path}: {timed(g):.2f} us  ({p.num_kernels} kernels, tile {p.describe()['tile']})")

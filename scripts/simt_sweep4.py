"""SIMT batched-layer sweep over lane-filling row-mode tiles (every lane of a
warp owns an output row: tn * th * groups a multiple of 32), timed with the
bench protocol (L2 flushed before each step, CUDA events around a graph
replay of conv_run), plus a relL2 check of the first two images against the
oracle.  One JSON line per tile."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs  # noqa: E402

dev = torch.device("cuda", 0)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
fw = torch.empty(2 * l2 // 4, device=dev)
fr = torch.ones_like(fw)
fo = torch.empty((), device=dev)


def timeit(plan, i, k, o, ws, n=10):
    st = torch.cuda.current_stream()
    s = torch.cuda.Stream()
    s.wait_stream(st)
    with torch.cuda.stream(s):
        plan.run(i, k, o, ws, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(i, k, o, ws, stream=s)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        fw.zero_()
        torch.sum(fr, dim=0, out=fo)
        a.record(st)
        g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ev])) * 1e3


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "batched"
    sh = CONFIGS[name]
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    ref = oracle.conv_eq1(xi.numpy()[:2], wi.numpy())
    specs = [None]
    for tk, tw in ((4, 14), (4, 7), (8, 7)):
        groups = (sh.W + tw - 1) // tw
        for th, tn, kg, bc in itertools.product((1, 2, 7, 14), (1, 2, 4, 8, 16, 32), (2, 4, 8, 16), (2, 4, 8)):
            slots = tn * th * groups
            if slots % 32 or slots > 128 or sh.H % th:
                continue
            pw = slots // 32
            if 32 * kg * pw > 512:
                continue
            specs.append(f"ver=2,tk={tk},tw={tw},kg={kg},pw={pw},tn={tn},th={th},bc={bc}")
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        except conv.ConvError as e:
            print(json.dumps({"spec": spec, "error": str(e)[:100]}), flush=True)
            continue
        o, ws = plan.new_output(), plan.new_workspace()
        us = timeit(plan, i, k, o, ws)
        got = o[:2].cpu().numpy().astype(np.float64)
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        d = plan.describe()
        print(json.dumps({"spec": spec, "tile": d["tile"], "us": round(us, 1), "tflops": round(sh.flops / us / 1e6, 2),
                          "model_us": round(d["model"]["model_us"], 1), "rel": rel}), flush=True)


if __name__ == "__main__":
    main()

"""Run one layer's plan a few times (for ncu captures): python scripts/run_layer.py NAME [path] [tile]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, TABLE1, make_inputs  # noqa: E402

name = sys.argv[1]
path = sys.argv[2] if len(sys.argv) > 2 else "bf16"
tile = sys.argv[3] if len(sys.argv) > 3 else None
sh = CONFIGS[name] if name in CONFIGS else TABLE1[name]
inp, ker = make_inputs(sh, seed=0)
plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile, **sh.plan_kwargs())
print(plan.describe()["tile"], flush=True)
i, k = inp.cuda(), ker.cuda()
out, ws = plan.new_output(), plan.new_workspace()
for _ in range(3):
    plan.run(i, k, out, ws)
torch.cuda.synchronize()

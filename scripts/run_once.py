"""Run one conv (path, config, optional tile) a few times: a small target for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
path, cfg = sys.argv[1], sys.argv[2]
tile = sys.argv[3] if len(sys.argv) > 3 else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
sh = CONFIGS[cfg]
plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile)
i, k = make_inputs(sh)
i, k = i.cuda(), k.cuda()
o = plan.new_output(); ws = plan.new_workspace()
for _ in range(reps):
    plan.run(i, k, o, ws)
torch.cuda.synchronize()
print(plan.describe()["tile"])

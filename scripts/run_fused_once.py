"""One fused conv_run on a config (experiments): prints ok or the error."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
path, cfg, tile = sys.argv[1], sys.argv[2], sys.argv[3]
sh = CONFIGS[cfg]
p = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile)
i, k = make_inputs(sh)
i, k = i.cuda(), k.cuda(); o = p.new_output(); ws = p.new_workspace()
try:
    for _ in range(2):
        p.run(i, k, o, ws)
    torch.cuda.synchronize()
    print("ok", p.describe()["tile"])
except Exception as e:
    print("FAIL", type(e).__name__, str(e)[:200])

"""Predicted strong-scaling efficiency of the batched layer from per-rank
shards timed on ONE GPU (the only kind this build can reach): for P in
{1, 2, 4, 8} the rank plan for N = 256/P images (shard.shard, the selector
re-tiles), timed with the bench protocol; efficiency = T1 / (P * TP).  The
ranks share nothing on the data path (non-reduction dims), so
the per-rank time is the multi-GPU step time up to the max-over-ranks
spread.  python scripts/shard_scaling_1gpu.py > profiles/.../shard_scaling.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, make_inputs  # noqa: E402
from paper_2101_09808_b200.shard import local_inputs, shard  # noqa: E402
from scripts.simt_sweep4 import timeit  # noqa: E402

full = CONFIGS["batched"]
inp, ker = make_inputs(full, seed=0)
for path in ("fp32_simt", "fp32_tc", "tf32", "bf16"):
    t1 = None
    for P in (1, 2, 4, 8):
        spec = shard(full, P, 0)
        li, lk = local_inputs(spec, inp, ker)
        plan = conv.ConvPlan(*spec.local.as_tuple(), path=path)
        i, k = li.cuda(), lk.cuda()
        o, ws = plan.new_output(), plan.new_workspace()
        us = timeit(plan, i, k, o, ws, n=20)
        t1 = t1 or us
        print(json.dumps({"path": path, "P": P, "per_rank_images": spec.local.N, "us": round(us, 2),
                          "tile": plan.describe()["tile"], "efficiency": round(t1 / (P * us), 3),
                          "aggregate_tflops": round(full.flops / us / 1e6, 1)}), flush=True)
        del i, k, o, ws
        torch.cuda.empty_cache()

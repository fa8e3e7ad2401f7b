"""The plans compute-sanitizer checks (memcheck / racecheck / synccheck, one
tool per gpurun call): the tiny and R2 layers on every path, a multi-wave
fused-transform plan (cross-CTA chunk flags), split-K plans (cross-CTA
arrival counters + TMA-staged reduction), a split-C SIMT plan and a
promoted FP32_TC plan.  Each runs twice; the two results must be
bit-identical (a race would show up here as well).

    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py [small]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import CONFIGS, Shape, make_inputs  # noqa: E402

CASES = [
    ("tiny", CONFIGS["tiny"], p, None) for p in ("fp32_simt", "fp32_tc", "tf32", "bf16")
] + [
    ("r2", CONFIGS["r2"], p, None) for p in ("fp32_simt", "fp32_tc", "tf32", "bf16")
] + [
    ("fused-2wave", Shape(N=160, K=256, C=256, H=14, W=14, R=3, S=3), "bf16", "fuse=1,cg=2"),
    ("fused-cg1", Shape(N=24, K=128, C=64, H=14, W=14, R=3, S=3), "tf32", "fuse=1,cg=1"),
    ("splitk-8", Shape.strided(1, 96, 320, 19, 17, 3, 3, 2, 2, 2, 1), "bf16", "splits=8"),
    ("splitk-3", Shape(N=1, K=128, C=256, H=7, W=7, R=3, S=3), "tf32", "splits=3"),
    ("simt-splitc", Shape(N=1, K=64, C=256, H=7, W=7, R=3, S=3), "fp32_simt", "splits=4"),
    ("fp32tc-promote", Shape(N=2, K=256, C=128, H=14, W=14, R=3, S=3), "fp32_tc", None),
]


def main():
    small = len(sys.argv) > 1 and sys.argv[1] == "small"
    torch.cuda.set_device(0)
    for name, sh, path, tile in CASES:
        if small and name.startswith("fused-2wave"):
            continue
        inp, ker = make_inputs(sh, seed=3)
        plan = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile, **sh.plan_kwargs())
        i, k = inp.cuda(), ker.cuda()
        a = plan.run(i, k)
        b = plan.run(i, k)
        torch.cuda.synchronize()
        same = torch.equal(a, b)
        print(f"{name:16s} {path:10s} {plan.describe()['tile']} deterministic={same}", flush=True)
        if not same:
            sys.exit(3)
    print("sanitize cases done")


if __name__ == "__main__":
    main()

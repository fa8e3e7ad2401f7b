"""Accumulation error of the tensor paths vs the length of the reduction:
relL2 against the oracle on the path's own (rounded / split) inputs, and
the mean signed error along sign(ref) (a negative mean = bias toward zero,
i.e. truncating accumulation).  FP32_TC (exact bf16 pieces) isolates the
tensor core's fp32 accumulation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2101_09808_b200 import conv  # noqa: E402
from paper_2101_09808_b200.inputs import Shape, make_inputs  # noqa: E402

tiles = sys.argv[1:] or [""]
for C in (16, 64, 256, 1024):
    sh = Shape(N=1, K=64, C=C, H=16, W=16, R=3, S=3)
    inp, ker = make_inputs(sh, seed=7)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy())
    for path, rnd in (("fp32_simt", lambda x: x), ("fp32_tc", lambda x: x), ("tf32", oracle.round_tf32_rna),
                      ("bf16", oracle.round_bf16_rne)):
        for tile in tiles if path == "fp32_tc" else [""]:
            p = conv.ConvPlan(*sh.as_tuple(), path=path, tile=tile or None)
            got = p.run(inp.cuda(), ker.cuda()).cpu().numpy().astype(np.float64)
            r = ref if path.startswith("fp32") else oracle.conv_eq1(rnd(inp.numpy()), rnd(ker.numpy()))
            d = got - r
            print(json.dumps({"C": C, "crs": 9 * C, "path": path, "tile": tile,
                              "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(r)),
                              "signed_bias": float(np.mean(d * np.sign(r)) / np.sqrt(np.mean(r * r)))}), flush=True)

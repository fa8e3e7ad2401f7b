"""Build an A/B variant of libconv.so from the same sources with extra nvcc
flags into _ab_<name>/libconv.so (git-ignored; it travels to the GPU box with
the snapshot).  Load it with CONV_LIB=_ab_<name>/libconv.so.

Usage: python scripts/build_ab.py NAME -DFLAG=1 [...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), f"_ab_{name}")
os.makedirs(out, exist_ok=True)
build._link(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), os.path.join(out, "libconv.so"),
            build.sources(), flags, False, f"ab_{name}")
print(os.path.join(out, "libconv.so"))

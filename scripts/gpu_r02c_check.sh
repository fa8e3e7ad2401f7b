#!/bin/bash
# r02c re-entry check on the GPU: the rebuilt tree's tests, smoke, default
# bench line and the reference arm
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_check
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"

#!/bin/bash
# fused (cooperative) In transform: parity first, then bench both ways
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_parity.py -x -q -k "fused" 2>&1 | tail -15 > gpurun_out/pytest_fused.log
cat gpurun_out/pytest_fused.log
for p in bf16 tf32; do
  for t in fuse=1 fuse=0; do
    timeout 300 python bench.py --path $p --tile $t --steps 30 --warmup 5 --soak 0.3 --no-cpu-baseline > gpurun_out/bench_${p}_$t.json 2> gpurun_out/bench_${p}_$t.err
    python -c "import json; d=json.load(open('gpurun_out/bench_${p}_$t.json')); print('$p $t', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_each'], d['config']['tile'], 'e2e', d['e2e']['value'])" || tail -5 gpurun_out/bench_${p}_$t.err
  done
  # transform alone: main kernel with no MMA / no TMA / no stores
  CONV_DEBUG_MODE=7 timeout 300 python bench.py --path $p --tile fuse=1 --steps 10 --warmup 3 --soak 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p transform-only kernel ms', d['roofline']['kernel_ms_each'])"
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log

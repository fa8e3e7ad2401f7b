#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_parity.py -x -q -k "fused" 2>&1 | tail -4
for t in fuse=1 fuse=0; do
  echo "== trace bf16 $t"; timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | tail -18
done
for p in bf16 tf32; do for t in fuse=1 fuse=0; do
  timeout 300 python bench.py --path $p --tile $t --steps 30 --warmup 5 --soak 0.3 --no-cpu-baseline > gpurun_out/bench_${p}_$t.json 2> gpurun_out/bench_${p}_$t.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${p}_$t.json')); print('$p $t', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_each'])" || tail -5 gpurun_out/bench_${p}_$t.err
done; done

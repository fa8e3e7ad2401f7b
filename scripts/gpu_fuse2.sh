#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in fuse=1 fuse=0; do
  echo "== trace bf16 $t"; timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | tail -16
done
echo "== transform only"
CONV_DEBUG_MODE=7 timeout 300 python bench.py --path bf16 --tile fuse=1 --steps 10 --warmup 3 --soak 0 --no-cpu-baseline > gpurun_out/dbg7.json 2> gpurun_out/dbg7.err; tail -3 gpurun_out/dbg7.err
python -c "import json; d=json.load(open('gpurun_out/dbg7.json')); print('transform-only kernel ms', d['roofline']['kernel_ms_each'])"
CONV_TRACE=/tmp/t7.bin CONV_DEBUG_MODE=7 timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | tail -8
timeout 600 python -m pytest tests/test_parity.py -x -q -k "fused or cta_group" 2>&1 | tail -4
for t in fuse=1 fuse=0; do
  timeout 300 python bench.py --path bf16 --tile $t --steps 30 --warmup 5 --soak 0.3 --no-cpu-baseline > gpurun_out/bench_bf16_$t.json 2> gpurun_out/bench_bf16_$t.err
  python -c "import json; d=json.load(open('gpurun_out/bench_bf16_$t.json')); print('bf16 $t', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_each'])" || tail -5 gpurun_out/bench_bf16_$t.err
done

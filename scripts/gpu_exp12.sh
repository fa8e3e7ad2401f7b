#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in 1 0; do
  echo "== korder(tap_outer)=$o"; CONV_KORDER=$o timeout 120 python scripts/quick_check.py bf16 batched 2>&1 | grep -E "kernel us|exact"
  CONV_KORDER=$o timeout 300 python bench.py --path bf16 --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  bench value', d['value'], 'step ms', d['ms_per_step'], 'kernels', d['roofline']['kernel_ms_each'])"
done
echo "== trace"; timeout 120 python scripts/trace_tc.py bf16 batched "" 2>&1 | tail -9
timeout 1200 python -m pytest tests/test_parity.py -x -q -k "tensor or p10 or p1 or p2" 2>&1 | tail -3

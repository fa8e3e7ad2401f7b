#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in 1 0; do for pdl in 0 1; do
  if [ $pdl = 1 ]; then export CONV_NO_PDL=1; else unset CONV_NO_PDL; fi
  echo "== korder(tap_outer)=$o no_pdl=$pdl"; CONV_KORDER=$o timeout 120 python scripts/quick_check.py bf16 batched 2>&1 | grep "kernel us"
  CONV_KORDER=$o timeout 300 python bench.py --path bf16 --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  bench value', d['value'], 'step ms', d['ms_per_step'], 'kernels', d['roofline']['kernel_ms_each'])"
done; done
unset CONV_NO_PDL
echo "== trace korder 1"; CONV_KORDER=1 timeout 120 python scripts/trace_tc.py bf16 batched "" 2>&1 | tail -9
echo "== trace korder 0"; CONV_KORDER=0 timeout 120 python scripts/trace_tc.py bf16 batched "" 2>&1 | tail -9

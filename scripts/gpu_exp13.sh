#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -3
for p in bf16 tf32; do for nt in 0 1; do
  if [ $nt = 1 ]; then export CONV_NO_TMA_REPACK=1; else unset CONV_NO_TMA_REPACK; fi
  echo "== $p no_tma_repack=$nt"
  timeout 300 python bench.py --path $p --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  bench value', d['value'], 'step ms', d['ms_per_step'], 'kernels', d['roofline']['kernel_ms_each'])"
done; done
unset CONV_NO_TMA_REPACK
for c in det r2 pw; do timeout 300 python bench.py --path bf16 --config $c --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  $c bench value', d['value'], 'step ms', d['ms_per_step'], 'kernels', d['roofline']['kernel_ms_each'])"; done

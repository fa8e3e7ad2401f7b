#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
CONV_PROLOGUE_C=256 timeout 300 python -m pytest tests/test_parity.py -x -q -k "fused" 2>&1 | tail -2
CONV_PROLOGUE_C=128 timeout 300 python -m pytest tests/test_parity.py -x -q -k "fused" 2>&1 | tail -2
for p in bf16 tf32; do for pc in 0 64 128 192 256; do
  CONV_PROLOGUE_C=$pc timeout 300 python bench.py --path $p --tile fuse=1 --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p pre_c=$pc', 'step_us', round(d['ms_per_step']*1e3,2), 'kernels_us', [round(x*1e3,2) for x in d['roofline']['kernel_ms_each']])" || echo "$p $pc FAILED"
done; done

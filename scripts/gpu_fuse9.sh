#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_parity.py -x -q -k "fused or cta_group" 2>&1 | tail -3
echo "== trace bf16 fuse=1"; timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | grep -v "^tile [3-9]\|effective\|CTAs traced\|tiles per" | tail -22
for c in batched det r2; do for p in bf16 tf32; do for t in fuse=0 fuse=1; do
  timeout 300 python bench.py --config $c --path $p --tile $t --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $p $t', 'step_us', round(d['ms_per_step']*1e3,2), 'kernels_us', [round(x*1e3,2) for x in d['roofline']['kernel_ms_each']])" || echo "$c $p $t FAILED"
done; done; done

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for dm in 0 256; do
  echo "== trace bf16 fuse=1 debug=$dm"; CONV_DEBUG_MODE=$dm timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | grep -v "^tile\|effective\|CTAs traced\|tiles per" | tail -12
  CONV_DEBUG_MODE=$dm timeout 300 python bench.py --path bf16 --tile fuse=1 --steps 30 --warmup 5 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_each'])"
done

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in "fuse=1" "fuse=1,kbs=1,stages=5" "fuse=1,kbs=1,stages=4" "fuse=1,kbs=2,stages=2" "fuse=0,kbs=1,stages=5" "fuse=0,kbs=1,stages=4" "fuse=0,kbs=2,stages=2"; do
  timeout 300 python bench.py --path bf16 --tile $t --steps 20 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['config']['tile'].get('tnb'), d['value'], d['ms_per_step'], d['roofline']['kernel_ms_each'])"
done

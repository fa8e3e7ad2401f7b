#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for dm in 0 64; do for t in fuse=0 fuse=1; do
  CONV_DEBUG_MODE=$dm timeout 300 python bench.py --path bf16 --tile $t --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('debug $dm $t', 'step_us', round(d['ms_per_step']*1e3,2), 'kernels_us', [round(x*1e3,2) for x in d['roofline']['kernel_ms_each']])"
done; done

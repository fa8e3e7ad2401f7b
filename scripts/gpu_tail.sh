#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for p in bf16 tf32; do for t in fuse=1 fuse=0; do for e in 0 1; do
  if [ $e = 1 ]; then export CONV_NO_TAIL_SPLIT=1; else unset CONV_NO_TAIL_SPLIT; fi
  timeout 300 python bench.py --path $p --tile $t --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p $t no_tail_split=$e', 'step_us', round(d['ms_per_step']*1e3,2), 'kernels_us', [round(x*1e3,2) for x in d['roofline']['kernel_ms_each']], d['value'])" || echo "$p $t FAILED"
done; done; done
unset CONV_NO_TAIL_SPLIT

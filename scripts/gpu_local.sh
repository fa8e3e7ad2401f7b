#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in tiny r2 pw det; do for p in bf16 tf32; do for t in fuse=0 fuse=2 auto; do
  tt=$t; if [ $t = auto ]; then tt=""; fi
  timeout 300 python bench.py --config $c --path $p ${tt:+--tile $tt} --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['config']['tile']; print('$c $p $t', 'step_us', round(d['ms_per_step']*1e3,2), 'fuse', t['fuse'], 'bn', t['bn'], 'cg', t['cg'], 'kbs', t['kbs'])" || echo "$c $p $t FAILED"
done; done; done

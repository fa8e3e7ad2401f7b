#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -3
for p in bf16 tf32; do
  timeout 300 python bench.py --path $p --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p value', d['value'], 'step us', round(d['ms_per_step']*1e3,2), 'e2e', d['e2e'])" || tail -3 /tmp/err.txt
done

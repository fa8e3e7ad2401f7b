#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -k "simt" 2>&1 | tail -2
for c in tiny r2 pw det batched; do
  timeout 300 python bench.py --config $c --path fp32_simt --steps 20 --warmup 3 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'step_us', round(d['ms_per_step']*1e3,2), 'TF/s', d['value'], 'frac', d['roofline']['frac'], d['config']['tile'])"
done

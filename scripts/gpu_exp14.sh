#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -3
for p in bf16 tf32 fp32_simt; do for c in batched det r2 pw tiny; do
  timeout 300 python bench.py --path $p --config $c --steps 20 --warmup 3 --soak 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p $c value', d['value'], 'step us', round(d['ms_per_step']*1e3,2), 'kernels us', [round(x*1e3,2) for x in d['roofline']['kernel_ms_each']], 'frac', d['roofline']['frac'], 'tile', d['config']['tile'])"
done; done

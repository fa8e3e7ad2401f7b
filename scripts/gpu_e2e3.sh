#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_parity.py -q -k "run_host" 2>&1 | tail -1
for c in 0 6; do
  CONV_HOST_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --soak 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c e2e', d['e2e']['ms_per_step'], d['e2e']['value'])"
done

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for c in 4 6 8; do
  CONV_HOST_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --soak 0 --no-cpu-baseline > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err; echo "rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); print('chunks $c e2e', d['e2e']['ms_per_step'])" || tail -5 gpurun_out/e2e_$c.err
done

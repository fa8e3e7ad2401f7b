#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
for c in tiny r2 det; do for p in bf16 tf32; do
  timeout 300 python bench.py --config $c --path $p --steps 30 --warmup 5 --soak 0.2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $p', 'step_us', round(d['ms_per_step']*1e3,2), d['config']['tile'])"
done; done
timeout 900 python bench.py --sweep table1 --path all --steps 20 --warmup 3 > gpurun_out/table1_v3.jsonl 2> gpurun_out/table1_v3.err; echo "sweep rc=$?"

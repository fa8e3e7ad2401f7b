#!/bin/bash
# r02e final verification on the GPU: tests, smoke, default bench line (kg=8
# flat tile + remainder launch on the device, kg=4 chunks in conv_run_host),
# reference arm, ncu launch list of the default bench command
cd "$(dirname "$0")/.."
O=gpurun_out/r02e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_default.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'])
for k,v in d.get('paths',{}).items(): print(k, v['value'], v['roofline']['frac'], v['clocks'].get('reasons'))"

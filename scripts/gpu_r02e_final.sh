#!/bin/bash
# r02e final verification on the GPU (6-channel chunks on the kg=8 flat tile,
# split-C remainder launch): tests, smoke, default bench line, reference arm,
# ncu launch list of the default bench command, --set full of the headline's
# grids, predicted strong scaling, Table-1 SIMT sweep
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/run_layer.py batched fp32_simt > $O/run_layer.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_direct_simt2 -c 2 -o $O/simt_bc6 python scripts/run_layer.py batched fp32_simt > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python scripts/shard_scaling_1gpu.py > $O/shard_scaling_1gpu.jsonl 2> $O/shard_scaling.err; echo "scaling rc=$?"
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_simt.jsonl 2> $O/t1_simt.err; echo "sweep rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_default.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'], d['config']['tile'])
for k,v in d.get('paths',{}).items(): print(k, v['value'], v['roofline']['frac'], v['clocks'].get('reasons'))
for l in open('$O/shard_scaling_1gpu.jsonl'):
    d=json.loads(l)
    if d['path']=='fp32_simt': t=d['tile']; print(d['P'], d['us'], d['efficiency'], {k:t[k] for k in ('kg','bc','splits','flat','rem')})"

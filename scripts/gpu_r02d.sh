#!/bin/bash
# r02d checkpoint on the GPU: tests, smoke, default bench line (flat SIMT tile
# with the remainder launch), the kg=4 flat tile for the e2e comparison,
# reference arm, ncu launch list of the default bench command, one --set full
# capture of the headline SIMT kernels, Table-1 SIMT sweep
cd "$(dirname "$0")/.."
O=gpurun_out/r02d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
for i in 1 2; do
timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/e2e_auto_$i.json 2>/dev/null
timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 --tile "flat=1,tk=4,kg=4,pw=1,bc=4" > $O/e2e_kg4_$i.json 2>/dev/null
timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 --tile "flat=1,tk=4,kg=4,pw=1,bc=4,rem=0" > $O/e2e_kg4_norem_$i.json 2>/dev/null
done
for f in $O/e2e_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], r['kernel_ms'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/run_layer.py batched fp32_simt > $O/run_layer.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_direct_simt2 -c 2 -o $O/simt_rem python scripts/run_layer.py batched fp32_simt > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_simt.jsonl 2> $O/t1_simt.err; echo "sweep rc=$?"

#!/bin/bash
# r02d: chunk depth / ring depth of the kg=8 flat tile with the remainder launch; e2e with the
# host pipeline's own (kg=4) tile; host-run parity
cd "$(dirname "$0")/.."
O=gpurun_out/r02d_bc
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "run_host or host_pipeline or remainder" > $O/pytest_host.log 2>&1; tail -1 $O/pytest_host.log
T="flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=8,pw=1,bc=6;flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=4,pw=1,bc=6"
for st in 2 3; do
CONV_SIMT_STAGES=$st timeout 600 python scripts/simt_sweep7.py batched 256,128 "$T" 2>&1 | sed "s/^/stages$st /" >> $O/bc_ab.txt
done
grep -o '^stages.*"N": [0-9]*.*"spec": "[^"]*".*"us": [0-9.]*\|error.*' $O/bc_ab.txt | sed 's/"tile".*"us"/us/; s/"tma": "on", //; s/{"config": "batched", //'
for i in 1 2; do
timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/e2e_auto_$i.json 2>/dev/null
done
for f in $O/e2e_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], r['kernel_ms'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done

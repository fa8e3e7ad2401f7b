#!/bin/bash
# r02c: e2e (conv_run_host) of the flat SIMT tile with the wave-aligned chunk
# plan vs the per-image tile; GPU tests after the FP32_TC compact default
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_e2e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/flat_plan_$i.json 2>/dev/null
  CONV_HOST_SPLIT=6,52,52,52,52,42 timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/flat_old_$i.json 2>/dev/null
  CONV_HOST_SPLIT=4,61,61,61,61,8 timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/flat_4_$i.json 2>/dev/null
  CONV_HOST_SPLIT=10,61,61,61,61,2 timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/flat_10_$i.json 2>/dev/null
  timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 --tile "ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8,flat=0" > $O/img_$i.json 2>/dev/null
  timeout 300 python bench.py --path fp32_tc --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/tc_$i.json 2>/dev/null
done
for f in $O/*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], r['kernel_ms'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done

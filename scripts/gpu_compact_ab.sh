#!/bin/bash
# r02c A/B: FP32_TC compact 3-piece workspace vs the 6-pair layout, and the
# e2e of the flat vs per-image SIMT tile, alternating in one box
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_ab
mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --path fp32_tc --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/tc_pairs_$i.json 2>/dev/null
  CONV_SPLIT_COMPACT=1 timeout 300 python bench.py --path fp32_tc --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/tc_compact_$i.json 2>/dev/null
  timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/simt_flat_$i.json 2>/dev/null
  timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 --tile "ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8,flat=0" > $O/simt_img_$i.json 2>/dev/null
done
for f in $O/*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], r['kernel_ms'], r.get('kernel_ms_each'), d['e2e']['value'], d['e2e']['ms_per_step'])"; done

#!/bin/bash
# r02e: explicit conv_run_host chunk plans (CONV_HOST_SPLIT) against the modeled one, FP32 SIMT batched layer
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_e2e
mkdir -p $O
for pass in 1 2; do
for sp in "" "7,61,61,61,40,20,6" "7,64,64,64,57" "7,64,64,64,37,20" "14,64,64,64,30,20" "7,64,64,64,30,20,7" "3,32,64,64,64,29" "7,32,64,64,64,25" "7,64,64,64,27,20,10"; do
  CONV_HOST_SPLIT=$sp timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/tmp.json')); print('$sp' or 'plan', d['e2e']['value'], d['e2e']['ms_per_step'])" | tee -a $O/e2e_splits.txt
done; done

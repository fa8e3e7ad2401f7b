#!/bin/bash
# r02c: conv_run_host chunk partitions with a tapered end (the last chunk's
# download is the exposed tail) on the flat SIMT plan
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_taper
mkdir -p $O
for sp in "7,61,61,61,61,5" "7,61,61,61,40,20,6" "7,61,61,50,40,25,12" "7,50,50,50,50,30,19" "4,30,61,61,61,30,9" "7,61,61,61,30,30,6" "12,61,61,61,40,21"; do
  CONV_HOST_SPLIT=$sp timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.3 --steps 30 > $O/s.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/s.json')); print('$sp', d['e2e']['value'], d['e2e']['ms_per_step'])" | tee -a $O/taper.txt
done

#!/bin/bash
# r02e: conv_run_host with two alternating compute streams for the FP32 SIMT chunks -- parity, fuzz, e2e A/B
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_twocomp
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "run_host or host" > $O/pytest_host.log 2>&1; tail -1 $O/pytest_host.log
for s in 31 33; do timeout 900 python scripts/fuzz_run_host.py 60 $s > $O/fuzz_run_host_$s.txt 2>&1; tail -1 $O/fuzz_run_host_$s.txt | cut -c1-300; done
for pass in 1 2 3; do
for one in "" 1; do
for sp in "" "7,61,61,61,40,20,6" "7,41,41,41,41,41,38,6" "7,30,30,30,30,30,30,30,30,9"; do
  if [ -z "$one" ]; then export CONV_HOST_TWO_COMP=1; else unset CONV_HOST_TWO_COMP; fi
  CONV_HOST_SPLIT=$sp timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 > $O/tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/tmp.json')); print('one_comp' if '$one' else 'two_comp', '$sp' or 'plan', d['e2e']['value'], d['e2e']['ms_per_step'])" | tee -a $O/e2e_ab.txt
done; done; done

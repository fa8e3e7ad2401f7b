#!/bin/bash
# r02b: SIMT model occupancy-efficiency study (v2 = FFMA2) on the Table-1 AUTO sweep
cd "$(dirname "$0")/.."
for cfg in "12 0.7" "8 1.0" "4 1.0" "6 0.85"; do
  set -- $cfg
  CONV_SIMT_EFF_WARPS=$1 CONV_SIMT_EFF_LONE=$2 timeout 300 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 2>/dev/null | sed "s/^/$1_$2 /"
done

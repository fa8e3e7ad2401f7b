#!/bin/bash
# r02b: SIMT model -- fractional (CTAs per SM) vs whole-wave time, Table-1 AUTO + shard sizes
cd "$(dirname "$0")/.."
for mode in frac whole; do
  if [ $mode = whole ]; then export CONV_SIMT_WHOLE_WAVES=1; else unset CONV_SIMT_WHOLE_WAVES; fi
  timeout 300 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 2>/dev/null | sed "s/^/$mode /"
  python scripts/simt_sweep7.py batched 32,64,128,256 "" 2>/dev/null | sed "s/^/$mode /"
done

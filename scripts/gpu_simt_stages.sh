#!/bin/bash
# r02b SIMT A/B: TMA ring depth x CTA shape (FFMA2, padding lanes fixed)
cd "$(dirname "$0")/.."
T="ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8;ver=2,tk=4,tw=14,kg=8,pw=1,tn=2,th=14,bc=8;ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=4;ver=2,tk=4,tw=14,kg=8,pw=1,tn=2,th=14,bc=4;ver=2,tk=4,tw=14,kg=2,pw=1,tn=2,th=14,bc=8;ver=2,tk=4,tw=14,kg=16,pw=1,tn=2,th=14,bc=4"
out=gpurun_out/sw7_stages.txt
: > $out
for st in 3 2 4; do
  CONV_SIMT_STAGES=$st python scripts/simt_sweep7.py batched 256 "$T" | sed "s/^/s$st /" >> $out 2>&1
done

#!/bin/bash
# r02b SIMT A/B: TMA padded vs flat lane-filling tiles, FFMA vs FFMA2, ring depth
cd "$(dirname "$0")/.."
P="ver=2,tk=4,tw=14,kg=8,pw=1,tn=2,th=14,bc=8;ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8"
F="ver=2,tk=4,tw=14,kg=1,pw=7,tn=16,th=14,bc=1;ver=2,tk=4,tw=14,kg=1,pw=7,tn=16,th=14,bc=2;ver=2,tk=4,tw=14,kg=2,pw=7,tn=16,th=14,bc=1;ver=2,tk=4,tw=14,kg=2,pw=7,tn=16,th=14,bc=2"
out=gpurun_out/sw7_flat.txt
: > $out
python scripts/simt_sweep7.py batched 256 ";$P;$F" | sed "s/^/ffma2 s3 /" >> $out 2>&1
CONV_SIMT_STAGES=4 python scripts/simt_sweep7.py batched 256 "$P;$F" | sed "s/^/ffma2 s4 /" >> $out 2>&1
CONV_SIMT_STAGES=2 python scripts/simt_sweep7.py batched 256 "$F" | sed "s/^/ffma2 s2 /" >> $out 2>&1
CONV_LIB=_ab_fma1/libconv.so python scripts/simt_sweep7.py batched 256 "$P;$F" | sed "s/^/ffma s3 /" >> $out 2>&1

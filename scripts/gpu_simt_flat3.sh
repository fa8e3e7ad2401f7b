#!/bin/bash
# r02c: flat row-mode SIMT tiles with 2-warp CTAs / 2-channel chunks (more
# resident CTAs, finer balance of the 7168 warp tasks over 148 SMs)
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_flat3
mkdir -p $O
T="ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8;flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=2,pw=1,bc=2;flat=1,tk=4,kg=4,pw=1,bc=2;flat=1,tk=4,kg=2,pw=2,bc=2;flat=1,tk=4,kg=1,pw=2,bc=2;flat=1,tk=4,kg=8,pw=1,bc=2"
for st in 2 3 4; do
CONV_SIMT_STAGES=$st timeout 900 python scripts/simt_sweep7.py batched 256,128 "$T" 2>&1 | sed "s/^/s$st /" >> $O/flat_ab.txt
done
grep -o '^s[0-9] .*"N": [0-9]*.*"spec": "[^"]*".*"us": [0-9.]*' $O/flat_ab.txt | sed 's/"tile".*"us"/us/; s/"tma": "on", //; s/{"config": "batched",//'

#!/bin/bash
# r02c: flat row-mode SIMT tiles with 3..6 k groups per CTA (CTA counts that
# balance over 148 SMs) vs the per-image row-mode tile
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_flat2
mkdir -p $O
timeout 600 python -m pytest tests/test_parity.py -m gpu -q -x -k "flat or tma_staging" > $O/pytest_flat.log 2>&1; tail -1 $O/pytest_flat.log
T="ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8;flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=5,pw=1,bc=4;flat=1,tk=4,kg=6,pw=1,bc=4;flat=1,tk=4,kg=3,pw=1,bc=4;flat=1,tk=4,kg=5,pw=1,bc=2;flat=1,tk=4,kg=5,pw=1,bc=8"
timeout 900 python scripts/simt_sweep7.py batched 256,128,64 "$T" > $O/flat_ab.txt 2>&1
timeout 300 python scripts/simt_sweep7.py batched 256,128,64,32 "" 2>&1 | sed "s/^/auto /" >> $O/flat_ab.txt
CONV_SIMT_STAGES=3 timeout 300 python scripts/simt_sweep7.py batched 256 "flat=1,tk=4,kg=5,pw=1,bc=4" 2>&1 | sed "s/^/s3 /" >> $O/flat_ab.txt
grep -o '"N": [0-9]*.*"spec": "[^"]*".*"us": [0-9.]*' $O/flat_ab.txt | sed 's/"tile".*"us"/us/; s/"tma": "on", //'

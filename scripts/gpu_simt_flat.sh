#!/bin/bash
# r02c: flat row-mode SIMT tiles (every lane an output row) vs the per-image
# row-mode tile on the batched layer, parity tests first
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_flat
mkdir -p $O
timeout 600 python -m pytest tests/test_parity.py -m gpu -q -x -k "flat or tma_staging" > $O/pytest_flat.log 2>&1; tail -3 $O/pytest_flat.log
T="ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8;flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=4,pw=2,bc=4;flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=2,pw=1,bc=4;flat=1,tk=4,kg=2,pw=2,bc=4;flat=1,tk=4,kg=4,pw=1,bc=8"
for st in 2 3; do
  CONV_SIMT_STAGES=$st timeout 600 python scripts/simt_sweep7.py batched 256,128 "$T" 2>&1 | sed "s/^/s$st /" >> $O/flat_ab.txt
done
timeout 300 python scripts/simt_sweep7.py batched 256 "" 2>&1 | sed "s/^/auto /" >> $O/flat_ab.txt
grep -o '"spec": "[^"]*".*"us": [0-9.]*' $O/flat_ab.txt | sed 's/"tile".*"us"/us/' | head -40

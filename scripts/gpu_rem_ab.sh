#!/bin/bash
# r02d: the flat tile's remainder launch -- parity tests, then A/B timing
cd "$(dirname "$0")/.."
O=gpurun_out/r02d_rem
mkdir -p $O
timeout 900 python -m pytest tests/test_parity.py -m gpu -q -x -k "remainder or flat_row or run_host_batched or p10 or simt" > $O/pytest_rem.log 2>&1; tail -3 $O/pytest_rem.log
T="flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=4,pw=1,bc=4,rem=0;flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=8,pw=1,bc=4,rem=0;flat=1,tk=4,kg=2,pw=1,bc=4;flat=1,tk=4,kg=2,pw=1,bc=4,rem=0;ver=2,tk=4,tw=14,kg=4,pw=1,tn=2,th=14,bc=8"
for i in 1 2; do
timeout 900 python scripts/simt_sweep7.py batched 256,128,64 "$T;" >> $O/rem_ab.txt 2>&1
done
grep -o '"N": [0-9]*.*"spec": "[^"]*".*"us": [0-9.]*\|error.*' $O/rem_ab.txt | sed 's/"tile".*"us"/us/; s/"tma": "on", //'

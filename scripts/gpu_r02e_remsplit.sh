#!/bin/bash
# r02e: the remainder launch with split-C -- parity (remainder tests), then the
# N = 32 / 64 shard tiles of the batched layer with and without it
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_remsplit
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "remainder or split" > $O/pytest_rem.log 2>&1; tail -1 $O/pytest_rem.log
T="flat=1,tk=4,kg=4,pw=1,bc=4,splits=2;flat=1,tk=4,kg=4,pw=1,bc=4,splits=2,rem=0;flat=1,tk=4,kg=8,pw=1,bc=4,splits=2;flat=1,tk=4,kg=8,pw=1,bc=4,splits=3;flat=1,tk=4,kg=4,pw=1,bc=4,splits=3;flat=1,tk=4,kg=8,pw=1,bc=4,splits=4;flat=1,tk=4,kg=4,pw=1,bc=8,splits=2;flat=0,tk=4,kg=4,splits=4;"
for i in 1 2; do
timeout 900 python scripts/simt_sweep7.py batched 32,64 "$T" > $O/shard_tiles_$i.txt 2>&1
grep -o '"N": [0-9]*.*"spec": "[^"]*"\|"rem": [0-9]\|"us": [0-9.]*\|error.*' $O/shard_tiles_$i.txt | paste - - - | head -40
done

#!/bin/bash
# r02e: 6-channel chunks on the flat kg=8 tile (2-deep ring), two alternating passes per batch size
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_bc6
mkdir -p $O
T256="flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=8,pw=1,bc=6;flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=8,pw=1,bc=6;flat=1,tk=4,kg=8,pw=1,bc=8"
timeout 900 python scripts/simt_sweep7.py batched 256,128 "$T256" > $O/bc6_big.txt 2>&1
T64="flat=1,tk=4,kg=8,pw=1,bc=4,splits=2;flat=1,tk=4,kg=8,pw=1,bc=6,splits=2;flat=1,tk=4,kg=4,pw=1,bc=4,splits=2;flat=1,tk=4,kg=4,pw=1,bc=6,splits=2;flat=1,tk=4,kg=8,pw=1,bc=4,splits=2;flat=1,tk=4,kg=8,pw=1,bc=6,splits=2"
timeout 900 python scripts/simt_sweep7.py batched 64,32 "$T64" > $O/bc6_small.txt 2>&1
for f in $O/bc6_big.txt $O/bc6_small.txt; do
grep -o '"N": [0-9]*.*"spec": "[^"]*"\|"rem": [0-9]\|"us": [0-9.]*\|error.*' $f | paste - - - ; done

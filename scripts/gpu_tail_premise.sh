#!/bin/bash
# r02d premise check for the SIMT tail plan: the flat tile at N = 253 (111 slot
# tiles x 16 k tiles = 1776 CTAs = 4 whole rounds of 3 x 148) against N = 256
# (1792), and unsplit tiles of a 3-image tail
cd "$(dirname "$0")/.."
O=gpurun_out/r02d_tail
mkdir -p $O
F="flat=1,tk=4,kg=4,pw=1,bc=4"
timeout 600 python scripts/simt_sweep7.py batched 256,253,252,222,148 "$F" > $O/main.txt 2>&1
T="ver=2,tk=4,tw=4,kg=4,pw=1,splits=1;ver=2,tk=4,tw=4,kg=2,pw=1,splits=1;ver=2,tk=4,tw=4,kg=1,pw=1,splits=1;ver=2,tk=8,tw=4,kg=2,pw=1,splits=1;ver=2,tk=8,tw=4,kg=1,pw=1,splits=1;ver=2,tk=4,tw=4,kg=4,pw=2,splits=1;ver=2,tk=4,tw=4,kg=2,pw=2,splits=1;ver=2,tk=4,tw=14,kg=4,pw=1,tn=1,th=14,splits=1;ver=2,tk=4,tw=14,kg=1,pw=1,tn=1,th=14,splits=1;ver=2,tk=4,tw=7,kg=1,pw=1,splits=1;ver=2,tk=4,tw=7,kg=2,pw=1,splits=1"
timeout 600 python scripts/simt_sweep7.py batched 3,4 "$T;" > $O/tail.txt 2>&1
grep -o '"N": [0-9]*.*"spec": "[^"]*".*"us": [0-9.]*\|error.*' $O/main.txt $O/tail.txt | sed 's/"tile".*"us"/us/; s/"tma": "on", //'

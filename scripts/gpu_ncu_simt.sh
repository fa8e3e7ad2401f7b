#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
C1="python scripts/run_once.py fp32_simt batched"
$C1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_direct -s 1 -c 1 -o gpurun_out/prof_simt_batched $C1 > gpurun_out/ncu_simt.log 2>&1; echo "rc=$?"
C2="python scripts/run_once.py fp32_simt batched ver=2,tk=8,tw=8,kg=4"
$C2 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_direct -s 1 -c 1 -o gpurun_out/prof_simt2_batched $C2 > gpurun_out/ncu_simt2.log 2>&1; echo "rc=$?"

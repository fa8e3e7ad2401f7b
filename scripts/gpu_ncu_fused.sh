#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
export CONV_NO_COOP=1
CMD="python bench.py --path bf16 --tile fuse=1 --steps 3 --warmup 3 --soak 0 --no-cpu-baseline --no-graph"
$CMD > gpurun_out/plain_fused.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 3 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_fused.log

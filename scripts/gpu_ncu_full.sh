#!/bin/bash
# ncu --set full of the default bench's main kernel and repack kernel (bf16 and tf32)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for p in bf16 tf32; do
  CMD="python bench.py --path $p --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-graph"
  $CMD > gpurun_out/plain_$p.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 3 -c 1 -o gpurun_out/prof_main_$p $CMD > gpurun_out/ncu_main_$p.log 2>&1
  echo "ncu main $p rc=$?"
  $CMD > gpurun_out/plain2_$p.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:repack -s 3 -c 1 -o gpurun_out/prof_repack_$p $CMD > gpurun_out/ncu_repack_$p.log 2>&1
  echo "ncu repack $p rc=$?"
done

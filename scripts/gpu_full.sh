#!/bin/bash
# GPU round: tests, bench, ncu launch list, ncu full capture of the main kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
for p in ${PATHS:-bf16 tf32}; do
  timeout 600 python bench.py --path $p --steps 20 --warmup 5 > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err; echo "bench $p rc=$?"; cat gpurun_out/bench_$p.json
done
if [ -n "$NCU" ]; then
  CMD="python bench.py --path bf16 --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
  echo "ncu list rc=$?"
  $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 3 -c 1 -o gpurun_out/prof_bf16 $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi

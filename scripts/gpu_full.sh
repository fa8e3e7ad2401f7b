#!/bin/bash
# GPU round: tests, smoke, bench (all paths), ncu launch list + full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for p in ${PATHS:-bf16 tf32 fp32_simt}; do
  timeout 900 python bench.py --path $p --steps 50 --warmup 5 > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err; echo "bench $p rc=$?"; cat gpurun_out/bench_$p.json
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
if [ -n "$NCU" ]; then
  CMD="python bench.py --path bf16 --steps 3 --warmup 3 --soak 0 --no-cpu-baseline"
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bf16.csv $CMD > gpurun_out/ncu_list.log 2>&1
  echo "ncu list rc=$?"
  $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 3 -c 1 -o gpurun_out/prof_bf16 $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
  C2="python scripts/run_once.py fp32_simt batched"
  $C2 > gpurun_out/plain3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_direct -s 1 -c 1 -o gpurun_out/prof_simt $C2 > gpurun_out/ncu_simt.log 2>&1
  echo "ncu simt rc=$?"
fi

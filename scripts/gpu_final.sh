#!/bin/bash
# consolidated GPU run: tests, smoke, default bench, reference arm, ncu launch list, Table-1 sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json
for p in tf32 fp32_simt; do
  timeout 600 python bench.py --path $p --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err; echo "bench $p rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 python bench.py --sweep table1 --path all --steps 20 --warmup 3 > gpurun_out/table1.jsonl 2> gpurun_out/table1.err; echo "sweep rc=$?"
# one full ncu capture of the headline main kernel per tensor path (roofline traffic, profiles/)
for p in bf16 tf32; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -c 1 -o gpurun_out/main_full_$p -f python scripts/run_layer.py batched $p > gpurun_out/ncu_full_$p.log 2>&1; echo "ncu full $p rc=$?"
done

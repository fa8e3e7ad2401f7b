#!/bin/bash
# r02c checkpoint on the GPU: tests, smoke, default bench line (flat SIMT
# headline tile), reference arm, ncu launch list of the default bench
# command, one --set full capture of the headline SIMT kernel
cd "$(dirname "$0")/.."
O=gpurun_out/r02c
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/run_layer.py batched fp32_simt > $O/run_layer.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_direct_simt2 -c 1 -o $O/simt_flat python scripts/run_layer.py batched fp32_simt > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_simt.jsonl 2> $O/t1_simt.err; echo "sweep rc=$?"

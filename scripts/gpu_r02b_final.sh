#!/bin/bash
# r02b final verification on the GPU: tests, smoke, default bench line (all
# paths), reference arm, ncu launch list of the default bench command,
# Table-1 SIMT sweep, predicted strong scaling from per-rank shards
cd "$(dirname "$0")/.."
O=gpurun_out/r02b_final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_simt.jsonl 2> $O/t1_simt.err; echo "sweep rc=$?"
timeout 600 python scripts/shard_scaling_1gpu.py > $O/shard_scaling_1gpu.jsonl 2> $O/shard_scaling.err; echo "shard rc=$?"

#!/bin/bash
# r02e (b): full GPU suite with the split-C remainder launch selected for the
# 32- / 64-image shards, predicted strong scaling, Table-1 SIMT sweep (unchanged picks)
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 600 python scripts/shard_scaling_1gpu.py > $O/shard_scaling_1gpu.jsonl 2> $O/shard_scaling.err; echo "scaling rc=$?"
python -c "
import json
for l in open('$O/shard_scaling_1gpu.jsonl'):
    d=json.loads(l); t=d['tile']; print(d['path'], d['P'], d['us'], d['efficiency'], d['aggregate_tflops'], {k:t[k] for k in t if k in ('tk','kg','bc','tn','flat','rem','splits','bm','bn','cg','fuse')})"
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_simt.jsonl 2> $O/t1_simt.err; echo "sweep rc=$?"

#!/bin/bash
# r02e: per-rank shard plans of the batched layer timed on one GPU (predicted
# strong scaling with the remainder launch), torchrun at world size 1, and the
# N = 32 / 64 SIMT tile candidates
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_scale
mkdir -p $O
timeout 600 python scripts/shard_scaling_1gpu.py > $O/shard_scaling_1gpu.jsonl 2> $O/shard_scaling.err; echo "scaling rc=$?"
python -c "
import json
for l in open('$O/shard_scaling_1gpu.jsonl'):
    d=json.loads(l); t=d['tile']; print(d['path'], d['P'], d['us'], d['efficiency'], d['aggregate_tflops'], {k:t[k] for k in t if k in ('tk','kg','bc','tn','flat','rem','splits','bm','bn','cg','fuse')})"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/torchrun_w1.json 2> $O/torchrun_w1.err; echo "torchrun rc=$?"
T="flat=1,tk=4,kg=8,pw=1,bc=4;flat=1,tk=4,kg=4,pw=1,bc=4;flat=1,tk=4,kg=4,pw=1,bc=4,splits=2;flat=1,tk=4,kg=8,pw=1,bc=4,splits=2;flat=1,tk=4,kg=2,pw=1,bc=4;flat=1,tk=4,kg=4,pw=1,bc=4,rem=0;flat=0,tk=4,kg=4,splits=2;flat=0,tk=4,kg=4,splits=4;flat=0,tk=8,kg=4,splits=2"
timeout 900 python scripts/simt_sweep7.py batched 64,32 "$T" > $O/shard_tiles.txt 2>&1
grep -o '"N": [0-9]*.*"spec": "[^"]*"\|"us": [0-9.]*\|error.*' $O/shard_tiles.txt | paste - - | head -40

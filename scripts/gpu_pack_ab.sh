#!/bin/bash
# r02c: tiled (transpose) SIMT Ker pack vs the per-element gather: GPU tests,
# Table-1 SIMT sweep and the batched bench line under both
cd "$(dirname "$0")/.."
O=gpurun_out/r02c_pack2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_tiled.jsonl 2> $O/t1_tiled.err; echo "sweep rc=$?"
CONV_SIMT_PACK_GATHER=0 timeout 900 python bench.py --sweep table1 --path fp32_simt --steps 10 --warmup 3 > $O/t1_alltiled.jsonl 2> $O/t1_alltiled.err; echo "sweep rc=$?"
for i in 1 2; do
  timeout 300 python bench.py --paths "" --no-cpu-baseline --no-e2e --soak 0.5 --steps 30 > $O/b_tiled_$i.json 2>/dev/null
  CONV_SIMT_PACK_GATHER=1 timeout 300 python bench.py --paths "" --no-cpu-baseline --no-e2e --soak 0.5 --steps 30 > $O/b_gather_$i.json 2>/dev/null
done
for f in $O/b_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], r['kernel_ms_each'])"; done
for f in $O/t1_*.jsonl; do python -c "
import json
t=p=0
for l in open('$f'):
  d=json.loads(l); t+=d['step_us']; p+=d['kernels_us'][0]
print('$f'.split('/')[-1], round(t,1), round(p,1))"; done

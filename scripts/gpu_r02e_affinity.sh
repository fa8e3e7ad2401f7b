#!/bin/bash
# r02e: e2e run-to-run spread (1.85 vs 2.1 ms on the same code) -- pinned buffers allocated from the GPU's local CPUs or not
cd "$(dirname "$0")/.."
O=gpurun_out/r02e_affinity
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; lscpu | grep -i "numa\|^CPU(s)\|Model name" >> $O/topo.txt; cat $O/topo.txt | head -20
for i in 1 2 3 4 5 6; do for a in gpu none; do
timeout 300 python bench.py --paths "" --no-cpu-baseline --soak 0.5 --steps 30 --cpu-affinity $a 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e'].get('host_buffers'))" | tee -a $O/affinity_ab.txt
done; done

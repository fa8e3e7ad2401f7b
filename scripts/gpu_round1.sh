#!/bin/bash
# first GPU contact: build, quick per-path checks (each in its own process)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for p in fp32_simt tf32 bf16; do
  for c in tiny r2 pw det batched; do
    timeout 120 python scripts/quick_check.py $p $c 2>&1 | tail -12
  done
done

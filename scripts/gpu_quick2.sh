#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for c in tiny r2 batched; do
  for t in "cg=2" "cg=1"; do
    timeout 120 python scripts/quick_check.py bf16 $c $t 2>&1 | tail -6
  done
done
for c in tiny r2 pw det batched; do timeout 120 python scripts/quick_check.py tf32 $c 2>&1 | tail -6; done
for c in tiny r2 pw det batched; do timeout 120 python scripts/quick_check.py bf16 $c 2>&1 | tail -6; done
for c in tiny r2 pw det batched; do timeout 120 python scripts/quick_check.py fp32_simt $c 2>&1 | tail -6; done

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
for m in 0 1 2 3 4 5 6 7; do
  for t in "cg=2" "cg=1" "cg=2,bn=128" "cg=1,bn=128"; do
    echo "mode=$m tile=$t"; CONV_DEBUG_MODE=$m timeout 120 python scripts/quick_check.py bf16 batched $t 2>&1 | grep "kernel us"
  done
done

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for f in 0 8 16; do
for m in 0 7 6; do
  for t in "cg=2" "cg=1" "cg=1,bn=128"; do
    echo "flavor=$f mode=$m tile=$t"; CONV_DEBUG_MODE=$((m+f)) timeout 120 python scripts/quick_check.py bf16 batched $t 2>&1 | grep -E "kernel us"
  done
done
done

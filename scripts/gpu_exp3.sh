#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for m in 0 7 6 5; do
  for t in "cg=2" "cg=1" "cg=1,bn=128" "cg=2,bn=128"; do
    echo "mode=$m tile=$t"; CONV_DEBUG_MODE=$m timeout 120 python scripts/quick_check.py bf16 batched $t 2>&1 | grep -E "kernel us|exact"
  done
done
for c in tiny r2 pw det batched; do timeout 120 python scripts/quick_check.py tf32 $c 2>&1 | tail -4; done

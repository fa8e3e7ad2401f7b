#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in "cg=2" "cg=1" "cg=1,bn=128"; do
  echo "== bf16 $t"; timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | tail -12
  echo "== bf16 mode6 $t"; CONV_DEBUG_MODE=6 timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | tail -12
done
echo "== tf32"; timeout 120 python scripts/trace_tc.py tf32 batched "" 2>&1 | tail -12

#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in "fuse=1" "fuse=0"; do
  for c in batched det r2; do echo "== bf16 $c [$t]"; timeout 120 python scripts/quick_check.py bf16 $c "$t" 2>&1 | tail -4; done
done
echo "== trace fused"; timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | tail -10
for t in "fuse=1" "fuse=0"; do echo "== tf32 batched [$t]"; timeout 120 python scripts/quick_check.py tf32 batched "$t" 2>&1 | tail -4; done
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -5

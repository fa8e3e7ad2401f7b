#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in "fuse=1" "fuse=0"; do
  for c in batched det; do echo "== bf16 $c [$t]"; timeout 120 python scripts/quick_check.py bf16 $c "$t" 2>&1 | tail -3; done
done
echo "== trace fused"; timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | tail -10
echo "== trace unfused"; timeout 120 python scripts/trace_tc.py bf16 batched "fuse=0" 2>&1 | tail -10
for t in "fuse=1" "fuse=0"; do echo "== tf32 batched [$t]"; timeout 120 python scripts/quick_check.py tf32 batched "$t" 2>&1 | tail -3; done
timeout 900 python scripts/simt_sweep.py det batched 2>&1 | grep -v infeasible
timeout 1200 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -3

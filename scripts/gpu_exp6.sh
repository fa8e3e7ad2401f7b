#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for t in "" "kbs=1" "cg=1,kbs=1" "cg=2,kbs=2,bn=128"; do
  echo "== bf16 [$t]"; timeout 120 python scripts/quick_check.py bf16 batched "$t" 2>&1 | tail -4
done
echo "== bf16 trace default"; timeout 120 python scripts/trace_tc.py bf16 batched "" 2>&1 | tail -9
for t in "" "kbs=1"; do echo "== tf32 [$t]"; timeout 120 python scripts/quick_check.py tf32 batched "$t" 2>&1 | tail -4; done
timeout 900 python -m pytest tests/test_parity.py -x -q -k "tensor or p10 or p1 or p2" 2>&1 | tail -5

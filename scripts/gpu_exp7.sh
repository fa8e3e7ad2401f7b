#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
./scripts/probe_mma; PROBE_RANDOM=1 ./scripts/probe_mma
for t in "" "kbs=1"; do echo "== bf16 trace [$t]"; timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | tail -10; done
echo "== tf32 trace"; timeout 120 python scripts/trace_tc.py tf32 batched "" 2>&1 | tail -10
timeout 900 python -m pytest tests/test_parity.py -x -q 2>&1 | tail -5

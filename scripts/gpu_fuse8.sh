#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
echo "== trace bf16 fuse=1"; timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | grep -v "^tile\|effective\|CTAs traced\|tiles per" | tail -18

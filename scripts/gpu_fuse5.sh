#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for dm in 0 7 1 2; do
  echo "== trace bf16 fuse=1 debug=$dm"; CONV_DEBUG_MODE=$dm timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | tail -14
done

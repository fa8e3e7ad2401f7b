#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for dm in 0 64 192; do
  echo "== trace bf16 fuse=1 debug=$dm"; CONV_DEBUG_MODE=$dm timeout 120 python scripts/trace_tc.py bf16 batched "fuse=1" 2>&1 | tail -17
done
for dm in 7 39; do for t in fuse=0 fuse=1; do
  echo "== debug $dm $t"; CONV_DEBUG_MODE=$dm timeout 120 python scripts/trace_tc.py bf16 batched "$t" 2>&1 | grep -E "Error|error|last epilogue|transform CTAs|end med"
done; done
timeout 600 python -m pytest tests/test_parity.py -x -q -k "fused or cta_group" 2>&1 | tail -4

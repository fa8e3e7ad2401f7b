#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
echo "debug2 fuse1:"; CONV_DEBUG_MODE=2 timeout 60 python scripts/run_fused_once.py bf16 batched fuse=1
echo "debug2 fuse1 nopdl:"; CONV_NO_PDL=1 CONV_DEBUG_MODE=2 timeout 60 python scripts/run_fused_once.py bf16 batched fuse=1
echo "debug2 fuse1 nocoop:"; CONV_NO_COOP=1 CONV_DEBUG_MODE=2 timeout 60 python scripts/run_fused_once.py bf16 batched fuse=1
echo "debug2 fuse1 cg1:"; CONV_DEBUG_MODE=2 timeout 60 python scripts/run_fused_once.py bf16 batched fuse=1,cg=1
echo "debug2 fuse1 r2:"; CONV_DEBUG_MODE=2 timeout 60 python scripts/run_fused_once.py bf16 r2 fuse=1
echo "debug2 fuse1 trace (no split):"; CONV_DEBUG_MODE=34 timeout 60 python scripts/run_fused_once.py bf16 batched fuse=1
echo "sanitizer debug2:"; CONV_DEBUG_MODE=2 timeout 300 compute-sanitizer --tool memcheck python scripts/run_fused_once.py bf16 r2 fuse=1 2>&1 | tail -25
echo "sanitizer normal:"; timeout 300 compute-sanitizer --tool memcheck python scripts/run_fused_once.py bf16 r2 fuse=1 2>&1 | tail -8

#!/bin/bash
# r02b: bf16 / tf32 batched -- the fused plan's prologue channels (pre_c) and stages
cd "$(dirname "$0")/.."
for t in "" "pre_c=0" "pre_c=64" "pre_c=128" "pre_c=256" "stages=4" "kbs=1,stages=6" "kbs=4,stages=2"; do
  for p in bf16 tf32; do
    v=$(timeout 120 python bench.py --path $p --paths "" --no-e2e --no-cpu-baseline --steps 30 --warmup 5 ${t:+--tile $t} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline']['step_frac'])")
    echo "$p ${t:-auto} $v"
  done
done

#!/bin/bash
# FP32_TC tile sweep on the batched layer (bench protocol); one JSON line per tile
out=${1:-gpurun_out/tc_sweep.jsonl}
for t in "bn=256,cg=2" "bn=192,cg=2" "bn=128,cg=2" "bn=256,cg=1" "bn=256,cg=2,kbs=1" "bn=256,cg=2,kbs=3" "bn=256,cg=2,split=9" "bn=128,cg=2,split=9"; do
  python bench.py --path fp32_tc --paths "" --tile "$t" --steps 10 --warmup 3 --soak 0.3 --no-cpu-baseline --no-e2e 2>>gpurun_out/tc_sweep.err | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(json.dumps({'tile_req':'$t','tile':j['config']['tile'],'value':j['value'],'kernel_ms':j['roofline']['kernel_ms'],'frac':j['roofline']['frac'],'ms':j['ms_per_step']}))" >> $out
done

#!/bin/bash
# r02e: model vs hardware counters for the FP32 SIMT path (Fig. 6 analog)
cd "$(dirname "$0")/.."
O=gpurun_out/fig6_simt
mkdir -p $O
M="dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,gpu__time_duration.sum"
run() {  # name layers stride
  timeout 300 python scripts/fig6_counters_simt.py run $2 $3 > $O/plain_$1.jsonl 2> $O/plain_$1.err || { echo "plain $1 failed"; tail -3 $O/plain_$1.err; return; }
  timeout 1500 ncu --metrics $M --clock-control none --csv --page raw --log-file $O/counters_$1.csv python scripts/fig6_counters_simt.py run $2 $3 > $O/manifest_$1.jsonl 2> $O/ncu_$1.err; echo "ncu $1 rc=$?"
  python scripts/fig6_counters_simt.py analyze $O/manifest_$1.jsonl $O/counters_$1.csv > $O/fig6_simt_$1.jsonl 2> $O/analyze_$1.err; echo "analyze $1 rc=$?"
  python -c "
import json
for l in open('$O/fig6_simt_$1.jsonl'):
    d=json.loads(l); print(d['layer'], d['tiles'], d['l2_smem'], d['hbm'], d['time'])"
}
run small r2,det,pw 1
run b64 batched64 3

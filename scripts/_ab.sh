for i in 1 2; do
  timeout 300 python bench.py --sweep table1 --path bf16 --steps 20 --warmup 3 > gpurun_out/ab7_cur_$i.jsonl 2>>gpurun_out/ab7.err
  timeout 300 python _ab_old/bench.py --sweep table1 --path bf16 --steps 20 --warmup 3 > gpurun_out/ab7_old_$i.jsonl 2>>gpurun_out/ab7.err
done
timeout 300 python bench.py --sweep table1 --path tf32 --steps 20 --warmup 3 > gpurun_out/ab7_tf32.jsonl 2>>gpurun_out/ab7.err

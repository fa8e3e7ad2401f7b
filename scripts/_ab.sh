for i in 1 2; do
  timeout 300 python bench.py --sweep table1 --path bf16 --steps 20 --warmup 3 > gpurun_out/ab6_cur_$i.jsonl 2>>gpurun_out/ab6.err
  timeout 300 python _ab_old/bench.py --sweep table1 --path bf16 --steps 20 --warmup 3 > gpurun_out/ab6_old_$i.jsonl 2>>gpurun_out/ab6.err
done

O=gpurun_out/r02t; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for D in 3 4 6; do for MS in 4096 8192 16384; do
  i=$((i+1))
  PAT_DEPTH=$D PAT_MIN_SLICE=$MS timeout 200 $R --master-port $((29750+i)) tools/zero3.py --caps 12,32 --iters 5 > $O/d${D}_ms${MS}.jsonl 2> $O/d${D}_ms${MS}.err
done; done

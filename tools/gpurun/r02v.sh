O=gpurun_out/r02v; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for SH in 25 50 90; do for P in 5 2; do
  i=$((i+1))
  PAT_PROTOCOL=$P PAT_POLL_SHARE=$SH timeout 200 $R --master-port $((29770+i)) tools/zero3.py --caps 12,32,64 --iters 5 > $O/p${P}_sh${SH}.jsonl 2> $O/p${P}_sh${SH}.err
done; done

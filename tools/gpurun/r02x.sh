O=gpurun_out/r02x; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29791 tools/zero3.py --caps 128,96 --iters 5 > $O/default.jsonl 2> $O/default.err
i=0
for PD in 2 3; do for SH in 75 90; do
  i=$((i+1))
  PAT_POLL_DEPTH=$PD PAT_POLL_SHARE=$SH timeout 200 $R --master-port $((29792+i)) tools/zero3.py --caps 12,32 --iters 5 > $O/pd${PD}_sh${SH}.jsonl 2> $O/pd${PD}_sh${SH}.err
done; done

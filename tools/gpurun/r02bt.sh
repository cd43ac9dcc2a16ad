O=gpurun_out/r02bt; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for N in 2 3 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --out $O/sweep_n${N}_graph.jsonl > $O/sweep_n${N}_graph.log 2>&1; echo "graph$N rc=$?" >> $O/rc.txt
done

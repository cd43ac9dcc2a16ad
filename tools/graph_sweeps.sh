# Latency sweeps, graph mode, torchrun one process per GPU, PAT vs NCCL Ring, n = 2, 3, 4.
export PAT_TIMEOUT_MS=10000
O=${O:-gpurun_out/final}; mkdir -p $O
for N in ${NS:-2 3 4}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --out $O/sweep_n${N}_graph.jsonl > $O/sweep_n${N}_graph.log 2>&1
  echo graph $N rc=$?
done
for N in ${BENCH_NS:-2 4}; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N > $O/bench$N.json 2> $O/bench$N.err; echo bench$N rc=$?
done

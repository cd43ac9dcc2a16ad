O=gpurun_out/r02bh; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for cfg in "PAT_THREADS=512 PAT_CHANNELS=148" "PAT_THREADS=256 PAT_CHANNELS=296" "PAT_THREADS=384 PAT_CHANNELS=148"; do
  tag=$(echo $cfg | tr ' =' '__')
  for N in 2 4; do
  env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2993$N \
    bench_sweep.py --mode loop --min-bytes 16777216 --max-bytes 1073741824 --dtypes f32 --iters 20 --no-nccl --out $O/l_${tag}_n$N.jsonl > $O/l_${tag}_n$N.log 2>&1
  env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2994$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 4194304 --dtypes f32 --no-nccl --out $O/g_${tag}_n$N.jsonl > $O/g_${tag}_n$N.log 2>&1
  done
done

O=gpurun_out/r02bd; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for CH in 128 148; do for N in 2 4; do
  PAT_CHANNELS=$CH timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2983$N \
    bench_sweep.py --mode graph --min-bytes 262144 --max-bytes 16777216 --dtypes f32 --no-nccl --out $O/g_ch${CH}_n$N.jsonl > $O/g_ch${CH}_n$N.log 2>&1
  PAT_CHANNELS=$CH timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2984$N \
    bench_sweep.py --mode loop --min-bytes 33554432 --max-bytes 1073741824 --dtypes f32 --iters 20 --no-nccl --out $O/l_ch${CH}_n$N.jsonl > $O/l_ch${CH}_n$N.log 2>&1
  PAT_CHANNELS=$CH timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2985$N bench.py --gpus $N --steps 20 --warmup 5 --no-nccl > $O/b_ch${CH}_n$N.json 2> $O/b_ch${CH}_n$N.err
done; done

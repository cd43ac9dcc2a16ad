# LL32 forced, graph mode, n = 2, 3, 4, 256 KiB - 32 MiB (multi-step range).
export PAT_TIMEOUT_MS=10000
O=${O:-gpurun_out/ll32}; mkdir -p $O
for N in ${NS:-2 3 4}; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2995$N \
    bench_sweep.py --mode graph --min-bytes 262144 --max-bytes 33554432 --dtypes f32 --protocol 5 --no-nccl \
    --out $O/n${N}${TAG}.jsonl > $O/n${N}${TAG}.log 2>&1
  echo ll32 $N rc=$?
done

# Loop-mode (bandwidth) sweep 8-64 MiB, n = 2, 3, 4, PAT vs NCCL Ring: the mid-size range where
# the cost model moves between LL32 and SIMPLE.
export PAT_TIMEOUT_MS=10000
O=${O:-gpurun_out/final}; mkdir -p $O
for N in ${NS:-2 3 4}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N \
    bench_sweep.py --mode loop --min-bytes 8388608 --max-bytes 67108864 --iters 20 --warmup 5 --dtypes f32 \
    --out $O/loopmid_n${N}.jsonl > $O/loopmid_n${N}.log 2>&1
  echo loop $N rc=$?
done

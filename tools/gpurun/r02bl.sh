O=gpurun_out/r02bl; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for N in 2 3 4; do for P in 1 5 2 0; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2998$N \
    bench_sweep.py --mode graph --min-bytes 8192 --max-bytes 16777216 --dtypes f32 --protocol $P --no-nccl \
    --out $O/n${N}_p${P}.jsonl > $O/n${N}_p${P}.log 2>&1
  echo "forced $N $P rc=$?" >> $O/rc.txt
done; done

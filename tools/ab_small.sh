export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/ab
for P in 5 1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes f32 --protocol $P --no-nccl \
    --out gpurun_out/ab/n2_p${P}.jsonl > gpurun_out/ab/n2_p${P}.log 2>&1
  echo ab $P rc=$?
done

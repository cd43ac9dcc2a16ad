export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ll128.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ll128.log
for N in 2 4; do for P in 1 4 2; do
  X=""; [ $P != 1 ] && X="--no-nccl"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench_sweep.py --mode graph --min-bytes 8192 --max-bytes 16777216 --dtypes f32 --protocol $P $X --out gpurun_out/ll128_n${N}_p${P}.jsonl > gpurun_out/ll128_n${N}_p${P}.log 2>&1; echo sweep $N $P rc=$?
done; done

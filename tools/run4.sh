export PAT_TIMEOUT_MS=5000
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4y.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu4y.log
for N in 4 3 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N > gpurun_out/bench${N}_v5.json 2> gpurun_out/bench${N}_v5.err; echo bench$N rc=$?
done
for N in 4 3 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench_sweep.py --mode graph --max-bytes 4194304 --dtypes f32 --out gpurun_out/sweep${N}_graph_v5.json > /dev/null 2>&1; echo sweepg$N rc=$?
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench_sweep.py --mode loop --min-bytes 8388608 --iters 10 --warmup 3 --out gpurun_out/sweep${N}_loop_v5.json > /dev/null 2>&1; echo sweepl$N rc=$?
done

export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench1 rc=$?
for N in 4 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N > gpurun_out/bench${N}.json 2> gpurun_out/bench${N}.err; echo bench$N rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench_sweep.py --mode loop --min-bytes 8388608 --iters 10 --warmup 3 --out gpurun_out/sweep4_loop.json > /dev/null 2>&1; echo sweepl4 rc=$?

export PAT_TIMEOUT_MS=5000
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu4.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1_v2.json 2>gpurun_out/bench1_v2.err; echo bench1 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench2_v2.json 2> gpurun_out/bench2_v2.err; echo bench2 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench_sweep.py --mode loop --out gpurun_out/sweep2_loop.json > gpurun_out/sweep2_loop.log 2>&1; echo sweep-loop rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench_sweep.py --mode graph --max-bytes 4194304 --dtypes f32 --out gpurun_out/sweep2_graph.json > gpurun_out/sweep2_graph.log 2>&1; echo sweep-graph rc=$?
timeout 300 python bench_sweep.py --mode loop --ranks 8 --out gpurun_out/sweep1_local8.json --max-bytes 268435456 --dtypes f32 > gpurun_out/sweep1_local8.log 2>&1; echo sweep-local rc=$?

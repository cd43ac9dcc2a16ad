export PAT_TIMEOUT_MS=5000
nvidia-smi topo -m > gpurun_out/topo4.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4x.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu4x.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench4 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench3 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench_sweep.py --mode graph --max-bytes 4194304 --out gpurun_out/sweep4_graph.json > gpurun_out/sweep4_graph.log 2>&1; echo sweep4g rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29515 bench_sweep.py --mode graph --max-bytes 4194304 --dtypes f32 --out gpurun_out/sweep3_graph.json > gpurun_out/sweep3_graph.log 2>&1; echo sweep3g rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench_sweep.py --mode loop --min-bytes 1048576 --out gpurun_out/sweep4_loop.json > gpurun_out/sweep4_loop.log 2>&1; echo sweep4l rc=$?

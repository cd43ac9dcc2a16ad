export PAT_TIMEOUT_MS=5000
timeout 300 python bench.py > gpurun_out/bench1_v4.json 2>gpurun_out/bench1_v4.err; echo bench1 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench2_v4.json 2> gpurun_out/bench2_v4.err; echo bench2 rc=$?
PAT_LL_THRESHOLD=8388608 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench_sweep.py --mode graph --min-bytes 65536 --max-bytes 8388608 --dtypes f32 --no-nccl --out gpurun_out/sweep2_graph_ll.json > gpurun_out/sweep2_graph_ll.log 2>&1; echo sweep-ll rc=$?

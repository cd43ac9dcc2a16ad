export PAT_TIMEOUT_MS=5000
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu5.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu5.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1_v3.json 2>gpurun_out/bench1_v3.err; echo bench1 rc=$?
timeout 300 python bench_sweep.py --mode graph --ranks 8 --out gpurun_out/sweep1_local8_graph.json --max-bytes 268435456 --dtypes f32,bf16 --iters 20 > gpurun_out/sweep1_local8.log 2>&1; echo sweep-local rc=$?
PAT_FUSED=-1 timeout 300 python bench_sweep.py --mode graph --ranks 8 --out gpurun_out/sweep1_local8_transport.json --max-bytes 268435456 --dtypes f32 --iters 20 > gpurun_out/sweep1_local8t.log 2>&1; echo sweep-local-t rc=$?

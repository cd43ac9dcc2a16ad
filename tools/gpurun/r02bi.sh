O=gpurun_out/r02bi; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for rep in 1 2; do for PT in 1 0; do for N in 2 4; do
  PAT_POLL_THREADS=$PT timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2995$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --no-nccl --out $O/g_pt${PT}_n${N}_$rep.jsonl > $O/g_pt${PT}_n${N}_$rep.log 2>&1
done; done; done
for PT in 1 0; do PAT_POLL_THREADS=$PT timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 4 --steps 20 --warmup 5 --no-nccl > $O/b4_pt$PT.json 2> $O/b4_pt$PT.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_integrity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

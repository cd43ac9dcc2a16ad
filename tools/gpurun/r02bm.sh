O=gpurun_out/r02bm; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for N in 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2999$N \
    bench_sweep.py --mode graph --min-bytes 65536 --max-bytes 1048576 --dtypes f32 --no-nccl --out $O/auto_n${N}.jsonl > $O/auto_n${N}.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

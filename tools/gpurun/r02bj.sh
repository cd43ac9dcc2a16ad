O=gpurun_out/r02bj; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for rep in 1 2; do for V in "" bars; do for N in 2 4; do
  PAT_LIB_VARIANT=$V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2996$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes f32 --no-nccl --out $O/g_${V:-new}_n${N}_$rep.jsonl > $O/g_${V:-new}_n${N}_$rep.log 2>&1
done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_integrity.py tests/test_gpu_stats.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

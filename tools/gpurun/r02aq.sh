O=gpurun_out/r02aq; mkdir -p $O
export PAT_TIMEOUT_MS=10000
for rep in 1 2; do for V in "" serialcred; do
  PAT_LIB_VARIANT=$V timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2990$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes f32 --no-nccl --out $O/n4_${V:-par}_$rep.jsonl > $O/n4_${V:-par}_$rep.log 2>&1
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

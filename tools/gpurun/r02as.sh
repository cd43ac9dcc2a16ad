O=gpurun_out/r02as; mkdir -p $O
export PAT_TIMEOUT_MS=10000
for rep in 1 2; do for V in "" prev; do for N in 2 4; do
  PAT_LIB_VARIANT=$V timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 262144 --dtypes f32 --colls ag --no-nccl --out $O/n${N}_${V:-new}_$rep.jsonl > $O/n${N}_${V:-new}_$rep.log 2>&1
done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "protocols_forced or local or misaligned or tails" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

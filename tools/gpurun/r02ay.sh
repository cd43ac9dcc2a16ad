O=gpurun_out/r02ay; mkdir -p $O
export PAT_TIMEOUT_MS=10000
for rep in 1 2; do for V in "" pollser; do for N in 2 4; do
  PAT_LIB_VARIANT=$V timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2997$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 4194304 --dtypes f32 --no-nccl --out $O/n${N}_${V:-new}_$rep.jsonl > $O/n${N}_${V:-new}_$rep.log 2>&1
done; done; done
for V in "" pollser; do PAT_LIB_VARIANT=$V timeout 300 python bench.py --gpus 4 --ranks 8 --steps 20 --warmup 5 > $O/sp8_${V:-new}.json 2> $O/sp8_${V:-new}.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_integrity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

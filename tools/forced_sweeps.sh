# Polling (LL, LL32) and SIMPLE forced, n = 2, 3, 4, graph mode: the calibration data of
# tools/fit_costmodel.py. PROTOS overrides the protocol list (default: 1 2 5).
export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/forced
for N in 2 3 4; do for P in ${PROTOS:-1 2 5}; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N \
    bench_sweep.py --mode graph --min-bytes 8192 --max-bytes 16777216 --dtypes f32 --protocol $P --no-nccl \
    --out gpurun_out/forced/n${N}_p${P}.jsonl > gpurun_out/forced/n${N}_p${P}.log 2>&1
  echo forced $N $P rc=$?
done; done
python tools/fit_costmodel.py gpurun_out/forced/*.jsonl --out gpurun_out/forced/fit.json | tail -14

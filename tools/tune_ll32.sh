# LL32 slot size (PAT_LL32_SLOT) at n = 4, forced LL32, graph mode, 256 KiB - 32 MiB.
export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/ll32slot
for S in ${SLOTS:-32768 65536 131072}; do
  PAT_LL32_SLOT=$S timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} --master-addr 127.0.0.1 --master-port 29931 \
    bench_sweep.py --mode graph --min-bytes 262144 --max-bytes 33554432 --dtypes f32 --protocol 5 --no-nccl \
    --out gpurun_out/ll32slot/s$S.jsonl > gpurun_out/ll32slot/s$S.log 2>&1
  echo slot $S rc=$?
done

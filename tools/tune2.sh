export PAT_TIMEOUT_MS=5000
for cfg in "64 262144 2 8" "96 262144 2 8" "128 131072 2 8" "128 262144 2 8" "64 524288 2 8" "96 131072 3 8" "128 262144 2 4" "64 262144 2 12"; do
  set -- $cfg
  tag="c$1_s$2_d$3_w$4"
  PAT_CHANNELS=$1 PAT_SLICE_BYTES=$2 PAT_DEPTH=$3 PAT_SEND_WARPS=$4 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench_sweep.py --out gpurun_out/tune3_$tag.json --min-bytes 1048576 --max-bytes 268435456 --dtypes f32 --no-nccl --iters 20 --warmup 5 > /dev/null 2>&1
  echo "$tag rc=$?"
done

# SIMPLE bandwidth knobs at 256 MiB / 1 GiB per rank, n=4 torchrun, loop mode.
export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/tune
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 \
    bench_sweep.py --mode loop --min-bytes 268435456 --max-bytes 1073741824 --iters 5 --warmup 2 --dtypes f32 --no-nccl \
    --out gpurun_out/tune/$tag.jsonl > gpurun_out/tune/$tag.log 2>&1
  echo $tag rc=$?; grep -h '"pat"' gpurun_out/tune/$tag.jsonl | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print('   ', r['coll'], r['bytes_per_rank'], round(r['busbw_gbs'], 1), 'slice', r['plan']['slice_bytes'], 'ch', r['plan']['channels'])"
}
run default
run slice512k PAT_SLICE_BYTES=524288
run slice256k PAT_SLICE_BYTES=262144
run sendw12 PAT_SEND_WARPS=12
run thr1024 PAT_THREADS=1024 PAT_SEND_WARPS=24
run ch64 PAT_CHANNELS=64 PAT_SLICE_BYTES=524288
run depth5 PAT_DEPTH=5

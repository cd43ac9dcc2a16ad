# SIMPLE mid-size knobs (4-64 MiB per rank), n=4 torchrun, loop + graph mode.
export PAT_TIMEOUT_MS=10000 PAT_LL_THRESHOLD=1
mkdir -p gpurun_out/tunemid
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29802 \
    bench_sweep.py --mode graph --min-bytes 4194304 --max-bytes 67108864 --iters 10 --warmup 3 --dtypes f32 --no-nccl \
    --out gpurun_out/tunemid/$tag.jsonl > gpurun_out/tunemid/$tag.log 2>&1
  echo $tag rc=$?; grep -h '"pat"' gpurun_out/tunemid/$tag.jsonl | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print('   ', r['coll'], r['bytes_per_rank'], round(r['us'], 1), round(r['busbw_gbs'], 1), 'slice', r['plan']['slice_bytes'], 'ch', r['plan']['channels'], 'it', r['plan']['iterations'])"
}
run default
run s32k PAT_SLICE_BYTES=32768
run s64k PAT_SLICE_BYTES=65536
run c64s64k PAT_CHANNELS=64 PAT_SLICE_BYTES=65536
run c64s128k PAT_CHANNELS=64 PAT_SLICE_BYTES=131072
run c32s128k PAT_CHANNELS=32 PAT_SLICE_BYTES=131072
run c96s48k PAT_CHANNELS=96 PAT_SLICE_BYTES=49152

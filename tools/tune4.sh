export PAT_TIMEOUT_MS=5000
timeout 600 python -m pytest tests -x -q -m gpu -k "multi_gpu or multiprocess or back_to_back or small_slots or protocols" > gpurun_out/pytest_gpu_skew2.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_skew2.log
for cfg in "128 0 1 0" "128 262144 1 0" "64 262144 1 2" "64 524288 1 2" "32 524288 1 2" "128 262144 0 2" "96 262144 1 0"; do
  set -- $cfg
  tag="c$1_s$2_k$3_d$4"
  if [ "$2" = "0" ]; then unset PAT_SLICE_BYTES; else export PAT_SLICE_BYTES=$2; fi
  if [ "$4" = "0" ]; then unset PAT_DEPTH; else export PAT_DEPTH=$4; fi
  PAT_CHANNELS=$1 PAT_SKEW=$3 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench_sweep.py --mode loop --out gpurun_out/tune4c_$tag.json --min-bytes 16777216 --max-bytes 536870912 --dtypes f32 --no-nccl --iters 10 --warmup 3 > gpurun_out/tune4c_$tag.log 2>&1
  echo "$tag rc=$?"
done

export PAT_TIMEOUT_MS=5000
timeout 600 python -m pytest tests -x -q -m gpu -k "multi_gpu or multiprocess or back_to_back or small_slots or protocols" > gpurun_out/pytest_gpu_skew.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_skew.log
for cfg in "0 1" "65536 1" "131072 1" "262144 1" "131072 0"; do
  set -- $cfg
  tag="s$1_k$2"
  if [ "$1" = "0" ]; then unset PAT_SLICE_BYTES; else export PAT_SLICE_BYTES=$1; fi
  PAT_SKEW=$2 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench_sweep.py --mode loop --out gpurun_out/tune4b_$tag.json --min-bytes 16777216 --max-bytes 536870912 --dtypes f32 --no-nccl --iters 10 --warmup 3 > gpurun_out/tune4b_$tag.log 2>&1
  echo "$tag rc=$?"
done

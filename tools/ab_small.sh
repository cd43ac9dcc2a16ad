# Small-message A/B at n = 2, graph mode: LL (1) and LL32 (5) forced, each with the knob in $AB
# (e.g. AB="PAT_PREFETCH=0 PAT_PREFETCH=1") set, on the same box.
export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/ab
for V in ${AB:-X=1}; do for P in 5 1; do
  env $V timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes f32 --protocol $P --no-nccl \
    --out gpurun_out/ab/n2_p${P}_${V}.jsonl > gpurun_out/ab/n2_p${P}_${V}.log 2>&1
  echo ab $V $P rc=$?
done; done

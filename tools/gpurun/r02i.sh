set -u
O=gpurun_out/r02i; mkdir -p $O
for cfg in "BENCH_SLEEP_CYCLES=200000" "BENCH_SLEEP_CYCLES=200000 BENCH_NO_CLOCKS=1" "BENCH_SLEEP_CYCLES=4000000" "BENCH_SLEEP_CYCLES=4000000 BENCH_NO_CLOCKS=1"; do
  for rep in 1 2; do
    tag=$(echo $cfg | tr ' =' '__')_$rep
    env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > $O/$tag.json 2> $O/$tag.err
  done
done

O=gpurun_out/r02k; mkdir -p $O
for i in 1 2 3 4; do
BENCH_TRIALS=6 BENCH_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2968$i bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > $O/b$i.json 2> $O/b$i.err
done

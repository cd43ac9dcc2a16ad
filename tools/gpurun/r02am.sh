O=gpurun_out/r02am; mkdir -p $O
for i in 1 2; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/b1_$i.json 2> $O/b1_$i.err; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29891 bench.py --gpus 2 --steps 20 --warmup 5 > $O/b2.json 2> $O/b2.err

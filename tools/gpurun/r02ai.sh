O=gpurun_out/r02ai; mkdir -p $O
PAT_HOST_PROFILE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 2 --steps 200 --warmup 5 --no-nccl > $O/b2.json 2> $O/b2.err
PAT_HOST_PROFILE=1 timeout 300 python bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu-baseline --no-extras > $O/b1.json 2> $O/b1.err

# N=8 torchrun rehearsal on a 4-GPU box: 8 processes, two per GPU (gloo for the handle exchange,
# no NCCL comparison); the driver's SCALE run takes this path on 8 GPUs
set -u
O=gpurun_out/r02bz; mkdir -p $O
export PAT_TIMEOUT_MS=30000
BENCH_SHARE_GPUS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29888 bench.py --gpus 8 --steps 20 --warmup 5 > $O/bench8_shared.json 2> $O/bench8_shared.err; echo "rc_b8=$?" >> $O/rc.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29889 bench.py --impl reference --gpus 8 --steps 20 --warmup 5 > $O/ref8.json 2> $O/ref8.err; echo "rc_ref8=$?" >> $O/rc.txt

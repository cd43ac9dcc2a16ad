# e2e with one H2D + one D2H copy per device per step (packed blocks): N=1, torchrun N=2, one-process N=2
set -u
O=gpurun_out/r02ca; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29862 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "rc_b2=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2_1p.json 2> $O/bench2_1p.err; echo "rc_b2_1p=$?" >> $O/rc.txt

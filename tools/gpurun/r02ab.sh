set -u
O=gpurun_out/r02ab; mkdir -p $O
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2983$N bench.py --gpus $N --steps 20 --warmup 5 > $O/bench$N.json 2> $O/bench$N.err; echo "rc_bench$N=$?" >> $O/rc.txt
done
PAT_TIMEOUT_MS=10000 timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc_pytest=$?" >> $O/rc.txt

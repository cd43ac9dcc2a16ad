# polling-path trace points: traces of the n=2 all-gather (8 B, 1 MiB), N=2 bench (no regression), parity
set -u
O=gpurun_out/r02ct; mkdir -p $O
for B in 8 1048576; do
  PAT_TRACE=8 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2990$((B % 7)) tools/trace_run.py --bytes $B --coll ag > $O/ag_$B.txt 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29862 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl --no-extras > $O/bench2.json 2> $O/bench2.err; echo "rc_b2=$?" >> $O/rc.txt
PAT_TIMEOUT_MS=10000 timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -m gpu -q -x > $O/parity.log 2>&1; echo "rc_parity=$?" >> $O/rc.txt

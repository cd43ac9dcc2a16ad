set -u
O=gpurun_out/r02b; mkdir -p $O
export BENCH_DEBUG=1
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > $O/b2_nonccl.json 2> $O/b2_nonccl.err
echo "rc_nonccl=$?" >> $O/rc.txt
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 2 --steps 20 --warmup 5 > $O/b2.json 2> $O/b2.err
echo "rc_nccl=$?" >> $O/rc.txt
timeout 300 ./tools/local_tune > $O/local_tune.jsonl 2> $O/local_tune.err
echo "rc_tune=$?" >> $O/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/rc.txt

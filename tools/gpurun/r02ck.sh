# tensor argument checks in the Python API: full GPU suite (2 GPUs), N=1 bench (eager cost), smoke
set -u
O=gpurun_out/r02ck; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 1200 python -m pytest tests -m gpu -q -x > $O/suite.log 2>&1; echo "rc_suite=$?" >> $O/rc.txt
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29862 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "rc_b2=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc_smoke=$?" >> $O/rc.txt

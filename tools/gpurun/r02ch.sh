# cross-stream ordering of transport calls: fixed build vs previous (oldord); full suite; N=2 bench
set -u
O=gpurun_out/r02ch; mkdir -p $O
export PAT_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_ordering.py -m gpu -q > $O/fixed.log 2>&1; echo "rc_fixed=$?" >> $O/rc.txt
PAT_LIB_VARIANT=oldord timeout 600 python -m pytest tests/test_gpu_ordering.py -m gpu -q > $O/old.log 2>&1; echo "rc_old=$?" >> $O/rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/suite.log 2>&1; echo "rc_suite=$?" >> $O/rc.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29862 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "rc_b2=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2_1p.json 2> $O/bench2_1p.err; echo "rc_b2_1p=$?" >> $O/rc.txt

set -u
O=gpurun_out/r02c; mkdir -p $O
timeout 300 ./tools/local_tune > $O/local_tune.jsonl 2> $O/local_tune.err; echo "rc_tune=$?" >> $O/rc.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 2 --steps 20 --warmup 5 > $O/b2.json 2> $O/b2.err; echo "rc_b2=$?" >> $O/rc.txt
for rep in 1 2; do for V in "" nohash; do
  PAT_LIB_VARIANT=$V timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2961$rep bench.py --gpus 2 --steps 200 --warmup 10 --no-nccl > $O/ab_${V:-hash}_$rep.json 2> $O/ab_${V:-hash}_$rep.err; echo "rc_ab_${V:-hash}_$rep=$?" >> $O/rc.txt
done; done
timeout 600 python -m pytest tests/test_gpu_multiprocess.py -x -q > $O/pytest_mp.log 2>&1; echo "pytest_mp_rc=$?" >> $O/rc.txt

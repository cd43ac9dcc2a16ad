# final library: GPU suite (4 GPUs), smoke, bench N=1 / torchrun N=2, N=4 / one-process N=2 / 8 ranks on 4 GPUs
set -u
O=gpurun_out/r02cr; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc_pytest=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc_smoke=$?" >> $O/rc.txt
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2986$N bench.py --gpus $N --steps 20 --warmup 5 > $O/bench$N.json 2> $O/bench$N.err; echo "rc_bench$N=$?" >> $O/rc.txt
done
timeout 300 python bench.py --gpus 4 --ranks 8 --steps 20 --warmup 5 > $O/bench4_r8_sp.json 2> $O/bench4_r8_sp.err; echo "rc_b4r8=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2_1p.json 2> $O/bench2_1p.err; echo "rc_b2_1p=$?" >> $O/rc.txt

# e2e host submission time per step; 3 vs 4 device buffer sets; torchrun N=2 and N=4
set -u
O=gpurun_out/r02cb; mkdir -p $O
export PAT_TIMEOUT_MS=10000
for N in 2 4; do
 for B in 3 4; do
  BENCH_E2E_BUFFERS=$B timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2986$N bench.py --gpus $N --steps 20 --warmup 5 --no-extras > $O/bench${N}_b$B.json 2> $O/bench${N}_b$B.err; echo "rc_b${N}_$B=$?" >> $O/rc.txt
 done
done
timeout 300 python bench.py --gpus 4 --ranks 8 --steps 20 --warmup 5 --no-extras > $O/bench4_r8.json 2> $O/bench4_r8.err; echo "rc_b4r8=$?" >> $O/rc.txt

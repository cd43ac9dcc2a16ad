set -u
O=gpurun_out/r02l; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 20 --warmup 5 > $O/bench$N.json 2> $O/bench$N.err; echo "rc_bench$N=$?" >> $O/rc.txt
done
for N in 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --algos pat,ring --out $O/ring_n${N}_graph.jsonl > $O/ring_n${N}.log 2>&1; echo "rc_ring$N=$?" >> $O/rc.txt
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N \
    bench_sweep.py --mode graph --min-bytes 16777216 --max-bytes 134217728 --dtypes f32 --iters 20 --out $O/mid_n${N}_graph.jsonl > $O/mid_n${N}.log 2>&1; echo "rc_mid$N=$?" >> $O/rc.txt
done
for W in "" "--windows"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 \
    bench_sweep.py --mode loop --min-bytes 4194304 --max-bytes 268435456 --dtypes bf16 --colls ag,rs --no-nccl $W --out $O/win${W:+1}_n4.jsonl > $O/win${W:+1}_n4.log 2>&1; echo "rc_win${W:+1}=$?" >> $O/rc.txt
done

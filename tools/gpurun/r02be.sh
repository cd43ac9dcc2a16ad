set -u
O=gpurun_out/r02be; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc_pytest=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc_smoke=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
for N in 2 4; do
  for rep in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2987$N bench.py --gpus $N --steps 20 --warmup 5 > $O/bench${N}_$rep.json 2> $O/bench${N}_$rep.err; echo "rc_bench${N}_$rep=$?" >> $O/rc.txt
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2988$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --out $O/sweep_n${N}_graph.jsonl > $O/sweep_n${N}.log 2>&1; echo "rc_sweep$N=$?" >> $O/rc.txt
done

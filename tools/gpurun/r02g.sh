set -u
O=gpurun_out/r02g; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/rc.txt
for C in 0 1; do
  PAT_COOP=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2960$C bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2_coop$C.json 2> $O/bench2_coop$C.err; echo "rc_bench2_coop$C=$?" >> $O/rc.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --algos pat,ring --out $O/ring_n2_graph.jsonl > $O/ring_n2_graph.log 2>&1; echo "rc_ring=$?" >> $O/rc.txt
for W in "" "--windows"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 \
    bench_sweep.py --mode loop --min-bytes 4194304 --max-bytes 268435456 --dtypes bf16 --colls ag,rs --no-nccl $W --out $O/win${W:+1}_n2.jsonl > $O/win${W:+1}_n2.log 2>&1; echo "rc_win${W:+1}=$?" >> $O/rc.txt
done

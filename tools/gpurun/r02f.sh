set -u
O=gpurun_out/r02f; mkdir -p $O
export PAT_TIMEOUT_MS=10000
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 20 --warmup 5 > $O/bench$N.json 2> $O/bench$N.err; echo "rc_bench$N=$?" >> $O/rc.txt
done
timeout 300 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4_sp.json 2> $O/bench4_sp.err; echo "rc_bench4_sp=$?" >> $O/rc.txt
for LF in 0 1; do
  PAT_LEAVES_FIRST=$LF timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$LF \
    bench_sweep.py --mode graph --min-bytes 1048576 --max-bytes 134217728 --dtypes f32 --colls ag --no-nccl --out $O/lf${LF}_n4.jsonl > $O/lf${LF}_n4.log 2>&1; echo "rc_lf$LF=$?" >> $O/rc.txt
done
for V in "" nohash; do
  PAT_LIB_VARIANT=$V timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29730 \
    bench_sweep.py --mode graph --min-bytes 524288 --max-bytes 16777216 --dtypes f32 --protocol 5 --no-nccl --out $O/ll32_${V:-hash}_n4.jsonl > $O/ll32_${V:-hash}_n4.log 2>&1; echo "rc_ll32_${V:-hash}=$?" >> $O/rc.txt
done

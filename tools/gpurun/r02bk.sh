O=gpurun_out/r02bk; mkdir -p $O
export PAT_TIMEOUT_MS=20000
for rep in 1 2; do for LF in 1 -1; do for N in 4 3; do
  if [ "$LF" = "-1" ]; then unset PAT_LEAVES_FIRST; else export PAT_LEAVES_FIRST=$LF; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2997$rep \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes f32 --no-nccl --out $O/g_lf${LF}_n${N}_$rep.jsonl > $O/g_lf${LF}_n${N}_$rep.log 2>&1
done; done; done

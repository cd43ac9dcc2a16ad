# Round-1 measurement set (run on a 4-GPU box). Outputs under gpurun_out/final/.
export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/final; rm -f gpurun_out/final/*
O=gpurun_out/final
timeout 900 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
# latency sweeps, graph mode, multi-process (torchrun) vs NCCL Ring
for N in 2 3 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N \
    bench_sweep.py --mode graph --min-bytes 8 --max-bytes 16777216 --dtypes f32 --out $O/sweep_n${N}_graph.jsonl > $O/sweep_n${N}_graph.log 2>&1
  echo graph $N rc=$?
done
# bandwidth sweeps, loop mode (L2 flushed per call), multi-process vs NCCL Ring
for N in 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N \
    bench_sweep.py --mode loop --min-bytes 8388608 --max-bytes 1073741824 --iters 10 --warmup 3 --dtypes ${LOOP_DTYPES:-f32,bf16} \
    --out $O/sweep_n${N}_loop.jsonl > $O/sweep_n${N}_loop.log 2>&1
  echo loop $N rc=$?
done
# single-process (one process drives every GPU) bandwidth
for G in 2 4; do
  timeout 300 python tools/sp_sweep.py --gpus $G --min-bytes 4194304 --max-bytes 1073741824 --out $O/sp_g${G}.jsonl > $O/sp_g${G}.log 2>&1
  echo sp $G rc=$?
done
# bench lines
timeout 300 python bench.py > $O/bench1.json 2> $O/bench1.err; echo bench1 rc=$?
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N > $O/bench$N.json 2> $O/bench$N.err; echo bench$N rc=$?
done
# ncu: launch list of the N=1 bench command, full set on the fused local kernels and on the
# transport kernel (local mode, LL at 1 MiB)
C="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 200 $C > $O/plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_local.csv $C > $O/ncu_l.log 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_ -s 40 -c 4 -o $O/prof_local_fused $C > $O/ncu_f.log 2>&1; echo ncu-full rc=$?
export PAT_FUSED=-1
timeout 200 $C > $O/plain_t.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pat_kernel -s 40 -c 2 -o $O/prof_local_transport $C > $O/ncu_t.log 2>&1; echo ncu-transport rc=$?

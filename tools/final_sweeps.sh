# The measurement set (run on a 4-GPU box): tests, smoke, sweeps vs NCCL, bench lines, ncu (HBM and
# NVLink), one-process latency for 2..8 ranks, eager C++ latency. Outputs under gpurun_out/final/.
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
unset PAT_FUSED
# NVLink counters of the multi-GPU transport kernel (one process, last device profiled)
G=$(python -c "import torch; print(min(torch.cuda.device_count(), 4))")
timeout 600 ncu --devices $((G-1)) --replay-mode application --clock-control none -k regex:pat_kernel \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file $O/ncu_nvlink_g$G.csv python tools/ncu_nvlink.py --gpus $G > $O/ncu_nvlink_g$G.log 2>&1; echo ncu-nvlink rc=$?
# one-process graph latency for 2..8 ranks (ranks share GPUs beyond the GPU count)
timeout 600 python tools/sp_graph.py --ranks 2,3,4,5,6,7,8 --out $O/sp_graph.jsonl > $O/sp_graph.log 2>&1; echo sp-graph rc=$?
# eager C-ABI latency from C++, launch threads off / on
g++ -O2 -std=c++17 tools/capi_latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_2506_20252_b200 -l:libpatb200.so \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$ORIGIN/../paper_2506_20252_b200' -o tools/capi_latency && \
  for T in 0 1; do PAT_LAUNCH_THREADS=$T timeout 60 tools/capi_latency $G 8 | sed "s/^/threads=$T /"; done > $O/capi_latency.txt 2>&1; echo capi rc=$?

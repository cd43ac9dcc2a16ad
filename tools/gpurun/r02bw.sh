O=gpurun_out/r02bw; mkdir -p $O
for cfg in "X=1" "PAT_LAUNCH_THREADS=0" "BENCH_E2E_BUFFERS=2"; do
  env $cfg timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > $O/b2sp_$(echo $cfg|tr '=' '_').json 2>/dev/null
done
timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 --no-group > $O/b2sp_nogroup.json 2>/dev/null

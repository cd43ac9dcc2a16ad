O=gpurun_out/r02bx; mkdir -p $O
for cfg in "PAT_WORKER_SPIN_US=2000" "PAT_WORKER_SPIN_US=100" "PAT_WORKER_SPIN_US=0" "PAT_LAUNCH_THREADS=0"; do
  for N in 2 4; do
  env $cfg timeout 300 python bench.py --gpus $N --steps 20 --warmup 5 --no-nccl > $O/b${N}sp_$(echo $cfg|tr '=' '_').json 2>/dev/null
  done
done

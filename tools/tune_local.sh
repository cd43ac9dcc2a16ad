# Launch shape of the fused single-device kernels (N=1 bench workload: 8 ranks, 1 MiB).
for X in 1 2 3 4 6 8; do
  PAT_LOCAL_CTAS_PER_SM=$X timeout 200 python bench.py --no-cpu-baseline --steps 2000 --warmup 20 > gpurun_out/local_$X.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/local_$X.json').read().strip().splitlines()[-1]); print('ctas/SM $X', round(d['value'],1), {k: round(v, 2) for k, v in d['latency_us'].items() if k != 'timing'})"
done

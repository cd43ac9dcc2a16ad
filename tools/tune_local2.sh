# Bulk-copy (TMA) all-gather vs the vector kernel, N=1 bench workload.
for T in 0 8192 16384 32768; do for X in 2 4 8; do
  PAT_LOCAL_TMA=$T PAT_LOCAL_CTAS_PER_SM=$X timeout 200 python bench.py --no-cpu-baseline --steps 2000 --warmup 20 > gpurun_out/localt_${T}_$X.json 2>gpurun_out/localt_${T}_$X.err
  python -c "import json; d=json.loads(open('gpurun_out/localt_${T}_$X.json').read().strip().splitlines()[-1]); print('tma $T ctas/SM $X', round(d['value'],1), {k: round(v, 2) for k, v in d['latency_us'].items() if k != 'timing'})" || tail -3 gpurun_out/localt_${T}_$X.err
done; done
# correctness of the TMA path: fused all-gather tests with the env set
PAT_LOCAL_TMA=16384 timeout 600 python -m pytest tests -q -x -m gpu -k "allgather or fused or misaligned or back_to_back" > gpurun_out/pytest_tma.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_tma.log

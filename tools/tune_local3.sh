for cfg in "8192 4 4" "8192 4 8" "8192 6 4" "8192 6 6" "4096 4 8" "4096 8 8" "12288 4 4" "16384 3 4" "6144 4 6"; do
  set -- $cfg
  PAT_LOCAL_TMA=$1 PAT_LOCAL_CTAS_PER_SM=$2 PAT_LOCAL_TMA_STAGES=$3 timeout 200 python bench.py --no-cpu-baseline --steps 2000 --warmup 20 > gpurun_out/lt3.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/lt3.json').read().strip().splitlines()[-1]); print('tile $1 ctas/SM $2 stages $3', round(d['value'],1), {k: round(v, 2) for k, v in d['latency_us'].items() if k != 'timing'})"
done

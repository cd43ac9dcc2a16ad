export PAT_TIMEOUT_MS=5000
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_suite6.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_suite6.log
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N > gpurun_out/bench${N}_c2.json 2> gpurun_out/bench${N}_c2.err; echo bench$N rc=$?
  python -c "import json; d=json.loads(open('gpurun_out/bench${N}_c2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['latency_us'], d['latency_floor'])"
done

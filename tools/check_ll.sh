export PAT_TIMEOUT_MS=5000
timeout 600 python tools/ll_stress.py > gpurun_out/ll_stress.log 2>&1; echo stress rc=$?; grep "bad$" gpurun_out/ll_stress.log
timeout 600 python tools/switch_stress.py > gpurun_out/switch_stress4.log 2>&1; echo sw rc=$?; grep "bad$" gpurun_out/switch_stress4.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_suite5.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_suite5.log
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N \
    bench_sweep.py --mode graph --min-bytes 65536 --max-bytes 8388608 --dtypes f32 --out gpurun_out/llsweep_n${N}.jsonl > /dev/null 2>&1
  echo graph $N rc=$?; python tools/show_sweep.py gpurun_out/llsweep_n${N}.jsonl
done

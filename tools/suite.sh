export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_suite$i.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_suite$i.log
done

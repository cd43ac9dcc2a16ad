export PAT_TIMEOUT_MS=5000
timeout 600 python tools/switch_stress.py > gpurun_out/switch_stress2.log 2>&1; echo rc=$?; grep "bad$" gpurun_out/switch_stress2.log
timeout 600 python tools/ll128_stress.py > gpurun_out/ll128_stress3.log 2>&1; echo stress rc=$?; grep "bad$" gpurun_out/ll128_stress3.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_suite3.log 2>&1; echo pytest-all rc=$?; tail -2 gpurun_out/pytest_suite3.log

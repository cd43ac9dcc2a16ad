export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
timeout 300 python tools/ll128_dbg.py > gpurun_out/ll128_dbg2.log 2>&1; echo dbg rc=$?; grep -c "bad bytes" gpurun_out/ll128_dbg2.log
timeout 600 python tools/ll128_stress.py > gpurun_out/ll128_stress2.log 2>&1; echo stress rc=$?; grep "bad$" gpurun_out/ll128_stress2.log
timeout 300 tools/bidir_probe 4 > gpurun_out/bidir4c.txt 2>&1; echo probe rc=$?; grep ce- gpurun_out/bidir4c.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all2.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_all2.log

export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
timeout 600 python tools/ll128_stress.py > gpurun_out/ll128_stress.log 2>&1; echo stress rc=$?; tail -8 gpurun_out/ll128_stress.log
timeout 300 tools/bidir_probe 4 > gpurun_out/bidir4b.txt 2>&1; echo probe rc=$?; grep ce- gpurun_out/bidir4b.txt

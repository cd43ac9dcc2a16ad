export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "pull or protocols or bulk" > gpurun_out/pytest_pull.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_pull.log
for G in 2 4; do for P in 2 3; do
timeout 300 python tools/sp_sweep.py --gpus $G --protocol $P --min-bytes 65536 --max-bytes 1073741824 --out gpurun_out/sp_pull.jsonl > gpurun_out/sp_$G_$P.log 2>&1; echo sp $G $P rc=$?
done; done

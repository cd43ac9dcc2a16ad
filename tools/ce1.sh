export PAT_TIMEOUT_MS=5000
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "copy_engine or bulk or switches" > gpurun_out/pytest_ce.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ce.log
for G in 2 4; do for P in 5 2; do
timeout 300 python tools/sp_sweep.py --gpus $G --protocol $P --min-bytes 4194304 --max-bytes 1073741824 --out gpurun_out/sp_ce.jsonl > gpurun_out/sp_ce_${G}_${P}.log 2>&1; echo sp $G $P rc=$?
done; done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_all.log

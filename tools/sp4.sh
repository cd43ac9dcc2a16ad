export PAT_TIMEOUT_MS=5000
timeout 200 python tools/sp_sweep.py --out gpurun_out/sp4_direct.json --min-bytes 1048576 > gpurun_out/sp4.log 2>&1; echo rc=$?
timeout 200 python tools/sp_sweep.py --out gpurun_out/sp4_staged.json --direct -1 --min-bytes 1048576 >> gpurun_out/sp4.log 2>&1; echo rc=$?
PAT_SLICE_BYTES=262144 timeout 200 python tools/sp_sweep.py --out gpurun_out/sp4_direct_s256.json --min-bytes 1048576 >> gpurun_out/sp4.log 2>&1; echo rc=$?
tail -3 gpurun_out/sp4.log

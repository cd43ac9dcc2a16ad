# cross-stream ordering: AG on stream A, RS on stream B, no sleep; fixed vs previous build
set -u
O=gpurun_out/r02ci; mkdir -p $O
export PAT_TIMEOUT_MS=3000
timeout 600 python -m pytest tests/test_gpu_ordering.py -m gpu -q > $O/fixed.log 2>&1; echo "rc_fixed=$?" >> $O/rc.txt
PAT_LIB_VARIANT=oldord timeout 900 python -m pytest tests/test_gpu_ordering.py -m gpu -q > $O/old.log 2>&1; echo "rc_old=$?" >> $O/rc.txt

# grouped pair with halves of different protocols: fixed build vs the previous build (oldgrp)
set -u
O=gpurun_out/r02cg; mkdir -p $O
export PAT_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_group.py -m gpu -q -k mixed > $O/fixed.log 2>&1; echo "rc_fixed=$?" >> $O/rc.txt
PAT_LIB_VARIANT=oldgrp timeout 600 python -m pytest tests/test_gpu_group.py -m gpu -q -k mixed -x > $O/old.log 2>&1; echo "rc_old=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_parity.py -m gpu -q -x > $O/group_parity.log 2>&1; echo "rc_suite=$?" >> $O/rc.txt

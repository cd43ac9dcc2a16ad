set -u
O=gpurun_out/r02n; mkdir -p $O
export PAT_TIMEOUT_MS=20000
PAT_LIB_VARIANT=bounds timeout 600 python tools/sanitize_run.py > $O/bounds_suite.log 2>&1; echo "rc_bounds_suite=$?" >> $O/rc.txt
PAT_LIB_VARIANT=bounds timeout 1200 python -m pytest tests -m gpu -x -q > $O/bounds_pytest.log 2>&1; echo "rc_bounds_pytest=$?" >> $O/rc.txt
CMD="python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "rc_ncu_launch=$?" >> $O/rc.txt
$CMD > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:local_ -s 6 -c 4 -o $O/prof_local $CMD > $O/ncu_full.log 2>&1; echo "rc_ncu_full=$?" >> $O/rc.txt

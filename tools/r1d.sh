export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/r1d
O=gpurun_out/r1d
timeout 900 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
timeout 300 python bench.py > $O/bench1.json 2> $O/bench1.err; echo bench1 rc=$?
C="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 200 $C > $O/plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_local.csv $C > $O/ncu_l.log 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_ -s 40 -c 4 -o $O/prof_local_fused $C > $O/ncu_f.log 2>&1; echo ncu-full rc=$?

export PAT_TIMEOUT_MS=5000
timeout 300 python bench.py > gpurun_out/bench1_v6.json 2> gpurun_out/bench1_v6.err; echo bench rc=$?
C="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 200 $C > gpurun_out/plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_local.csv $C > gpurun_out/ncu_l.log 2>&1; echo ncu-launch rc=$?
timeout 200 $C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_ -s 40 -c 4 -o gpurun_out/prof_local_fused $C > gpurun_out/ncu_f.log 2>&1; echo ncu-full rc=$?
export PAT_FUSED=-1
timeout 200 $C > gpurun_out/plain_t.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pat_kernel -s 40 -c 2 -o gpurun_out/prof_local_transport $C > gpurun_out/ncu_t.log 2>&1; echo ncu-transport rc=$?

set -u
O=gpurun_out/r02af; mkdir -p $O
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
CMD="python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
$CMD > $O/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:local_group -s 3 -c 3 -o $O/prof_group $CMD > $O/ncu_full.log 2>&1; echo "rc_ncu=$?" >> $O/rc.txt
$CMD > $O/plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "rc_ncu2=$?" >> $O/rc.txt

O=gpurun_out/r02bc; mkdir -p $O
for N in 2 4; do
CMD="python tools/ncu_nvlink.py --gpus $N --cases grp:1048576,ag:1048576,rs:1048576"
PAT_LAUNCH_THREADS=0 $CMD > $O/plain$N.log 2>&1 && PAT_LAUNCH_THREADS=0 ncu --devices $((N-1)) --replay-mode application --clock-control none -k regex:pat_ --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $O/ncu_nvlink_g$N.csv $CMD > $O/ncu$N.log 2>&1; echo "rc$N=$?" >> $O/rc.txt
done

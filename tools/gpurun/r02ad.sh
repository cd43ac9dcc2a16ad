O=gpurun_out/r02ad; mkdir -p $O
CMD="python tools/ncu_nvlink.py --gpus 2 --cases ag:1048576,rs:1048576,ag:268435456,rs:268435456"
PAT_LAUNCH_THREADS=0 $CMD > $O/plain.log 2>&1 && PAT_LAUNCH_THREADS=0 ncu --devices 1 --replay-mode application --clock-control none -k regex:pat_kernel --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $O/ncu_nvlink_g2.csv $CMD > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log

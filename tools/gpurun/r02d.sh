set -u
O=gpurun_out/r02d; mkdir -p $O
timeout 300 ./tools/local_tune > $O/local_tune.jsonl 2> $O/local_tune.err; echo "rc_tune=$?" >> $O/rc.txt
timeout 200 python tools/eager_probe.py > $O/eager_probe.json 2> $O/eager_probe.err; echo "rc_eager=$?" >> $O/rc.txt
timeout 200 ./tools/capi_latency 1 1048576 > $O/capi.txt 2>&1; echo "rc_capi=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 1 --steps 400 --warmup 5 --no-cpu-baseline > $O/bench1_k400.json 2> $O/bench1_k400.err; echo "rc_b1k=$?" >> $O/rc.txt

O=gpurun_out/r02bs; mkdir -p $O
export PAT_TIMEOUT_MS=20000
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 3 --steps 20 --warmup 5 > $O/bench3.json 2> $O/bench3.err; echo "rc_b3=$?" >> $O/rc.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29732 \
  bench_sweep.py --mode graph --min-bytes 8 --max-bytes 1048576 --dtypes i32 --out $O/sweep_n3_i32.jsonl > $O/sweep_n3_i32.log 2>&1; echo "rc_sw=$?" >> $O/rc.txt

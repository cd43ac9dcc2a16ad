export PAT_TIMEOUT_MS=10000
mkdir -p gpurun_out/r1e
O=gpurun_out/r1e
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref1.json 2> $O/ref1.err; echo ref1 rc=$?; cat $O/ref1.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > $O/ref2.json 2> $O/ref2.err; echo ref2 rc=$?; cat $O/ref2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29732 tools/zero3.py --caps 512,256,128,64 > $O/zero3_n4.jsonl 2> $O/zero3_n4.err; echo zero3 rc=$?; cat $O/zero3_n4.jsonl
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29733 \
    bench_sweep.py --mode loop --min-bytes 8388608 --max-bytes 1073741824 --iters 10 --warmup 3 --dtypes f32,bf16 \
    --out $O/sweep_n3_loop.jsonl > $O/sweep_n3_loop.log 2>&1; echo loop3 rc=$?
python tools/show_sweep.py $O/sweep_n3_loop.jsonl

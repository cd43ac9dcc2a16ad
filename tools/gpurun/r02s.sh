O=gpurun_out/r02s; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
PAT_TRACE=1024 timeout 200 $R --master-port 29741 tools/trace_run.py --bytes 67108864 --coll rs --dtype bf16 --staging-mib 12 > $O/rs_12.txt 2>&1
PAT_TRACE=1024 timeout 200 $R --master-port 29742 tools/trace_run.py --bytes 67108864 --coll rs --dtype bf16 --staging-mib 0 > $O/rs_0.txt 2>&1
PAT_TRACE=1024 timeout 200 $R --master-port 29743 tools/trace_run.py --bytes 67108864 --coll ag --dtype bf16 --staging-mib 12 > $O/ag_12.txt 2>&1

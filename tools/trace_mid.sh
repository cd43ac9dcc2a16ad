export PAT_TIMEOUT_MS=5000 PAT_TRACE=256 PAT_LL_THRESHOLD=1
for b in 16777216 67108864; do for c in ag rs; do
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29700 tools/trace_run.py --bytes $b --coll $c > gpurun_out/trace4_${c}_$b.txt 2>&1; echo $c $b rc=$?
cat gpurun_out/trace4_${c}_$b.txt | grep -v "^\[\|NCCL\|W10\|warn"
done; done

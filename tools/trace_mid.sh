# Device event traces of mid-size SIMPLE calls at n = 4 (torchrun), rank 0 timeline summaries.
export PAT_TIMEOUT_MS=5000 PAT_TRACE=256 PAT_LL_THRESHOLD=1 PAT_PROTOCOL=2
for b in ${SIZES:-4194304 16777216}; do for c in ${COLLS:-ag rs}; do
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29700 tools/trace_run.py --bytes $b --coll $c > gpurun_out/trace4_${c}_$b.txt 2>&1; echo $c $b rc=$?
cat gpurun_out/trace4_${c}_$b.txt | grep -v "^\[\|NCCL\|W10\|warn"
done; done

export PAT_TIMEOUT_MS=10000 PAT_TRACE=256
for b in 268435456; do for c in ag rs; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 tools/trace_run.py --bytes $b --coll $c > gpurun_out/traceb_${c}_$b.txt 2>&1; echo $c $b rc=$?
python tools/fence_cost.py gpurun_out/trace_${c}_${b}_r0.npz gpurun_out/trace_${c}_${b}_r1.npz
done; done

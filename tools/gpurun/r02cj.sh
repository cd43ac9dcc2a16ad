# eager cost of the cross-stream ordering event: same box, previous build (oldord) vs current, N=2 torchrun, 2 repeats
set -u
O=gpurun_out/r02cj; mkdir -p $O
for rep in 1 2; do
 for V in oldord cur; do
  if [ $V = cur ]; then unset PAT_LIB_VARIANT; else export PAT_LIB_VARIANT=$V; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2986$rep bench.py --gpus 2 --steps 20 --warmup 5 --no-extras --no-nccl > $O/b2_${V}_$rep.json 2> /dev/null; echo "rc_${V}_$rep=$?" >> $O/rc.txt
 done
done
unset PAT_LIB_VARIANT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29869 tools/eager_probe_mp.py > $O/probe_cur.txt 2>&1
PAT_LIB_VARIANT=oldord timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29870 tools/eager_probe_mp.py > $O/probe_old.txt 2>&1

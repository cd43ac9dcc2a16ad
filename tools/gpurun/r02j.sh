O=gpurun_out/r02j; mkdir -p $O
for i in 1 2 3; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2968$i tools/step_probe.py --sets 42 >> $O/probe42.txt 2>&1
PAT_POLL_DEPTH=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2969$i tools/step_probe.py --sets 42 >> $O/probe42_d3.txt 2>&1
done

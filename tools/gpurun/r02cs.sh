# device trace (CTA start/end) of the 1 MiB and 8-byte LL32 / auto all-gather at n=2
set -u
O=gpurun_out/r02cs; mkdir -p $O
for B in 8 1048576; do
  PAT_TRACE=8 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2990$((B % 7)) tools/trace_run.py --bytes $B --coll ag > $O/ag_$B.txt 2>&1
done

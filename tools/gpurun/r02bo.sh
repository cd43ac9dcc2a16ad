O=gpurun_out/r02bo; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for G in "" "--group"; do for W in "" "--windows"; do
  timeout 400 $R --master-port 29701 tools/zero3.py --caps 0,12 $G $W > $O/z${G:+g}${W:+w}.jsonl 2> $O/z${G:+g}${W:+w}.err
done; done

O=gpurun_out/r02bg; mkdir -p $O
export NCCL_ALGO=Ring
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 $R --master-port 29991 tools/zero3.py --caps 0,128,64,32,12 --nccl > $O/zero3_n4.jsonl 2> $O/zero3_n4.err
timeout 400 $R --master-port 29992 tools/zero3.py --caps 0,32,12 --windows > $O/zero3_win_n4.jsonl 2> $O/zero3_win_n4.err

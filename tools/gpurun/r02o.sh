set -u
O=gpurun_out/r02o; mkdir -p $O
export NCCL_ALGO=Ring
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 tools/zero3.py --caps 0,512,128,64,32,12 --nccl > $O/zero3_n4.jsonl 2> $O/zero3_n4.err; echo "rc=$?" >> $O/rc.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 tools/zero3.py --caps 0,512,128,64,32,12 --windows > $O/zero3_win_n4.jsonl 2> $O/zero3_win_n4.err; echo "rc_win=$?" >> $O/rc.txt

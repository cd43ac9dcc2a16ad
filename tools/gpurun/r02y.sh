O=gpurun_out/r02y; mkdir -p $O
export NCCL_ALGO=Ring
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 $R --master-port 29781 tools/zero3.py --caps 0,512,128,64,32,12 --nccl > $O/zero3_n4.jsonl 2> $O/zero3_n4.err
timeout 400 $R --master-port 29782 tools/zero3.py --caps 0,512,128,64,32,12 --windows > $O/zero3_win_n4.jsonl 2> $O/zero3_win_n4.err
PAT_TIMEOUT_MS=10000 timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log

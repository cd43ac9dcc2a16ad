set -u
O=gpurun_out/r02p; mkdir -p $O
export NCCL_ALGO=Ring
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29711 tools/zero3.py --caps 0,32,12 --windows > $O/win.jsonl 2> $O/win.err
for D in 4 6 8; do
  PAT_DEPTH=$D timeout 300 $R --master-port 2972$D tools/zero3.py --caps 32,12 > $O/depth$D.jsonl 2> $O/depth$D.err
done
for MS in 8192 16384 65536; do
  PAT_MIN_SLICE=$MS timeout 300 $R --master-port 29731 tools/zero3.py --caps 32,12 > $O/minslice$MS.jsonl 2> $O/minslice$MS.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_parity.log

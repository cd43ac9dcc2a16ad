O=gpurun_out/r02bf; mkdir -p $O
for rep in 1 2; do for NB in 2 3; do
BENCH_E2E_BUFFERS=$NB timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2989$rep bench.py --gpus 4 --steps 20 --warmup 5 --no-nccl > $O/b4_nb${NB}_$rep.json 2> $O/b4_nb${NB}_$rep.err
done; done
timeout 100 python tools/pcie_probe.py > $O/pcie.json 2>&1

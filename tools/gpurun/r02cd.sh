# e2e A/B on one box: N=1 and one-process N=2 with 3 vs 4 device sets, each twice
set -u
O=gpurun_out/r02cd; mkdir -p $O
export PAT_TIMEOUT_MS=10000
for rep in 1 2; do
 for B in 3 4; do
  BENCH_E2E_BUFFERS=$B timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-extras > $O/bench1_b${B}_$rep.json 2> /dev/null; echo "rc=$?" >> $O/rc.txt
  BENCH_E2E_BUFFERS=$B timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 --no-extras > $O/bench2_1p_b${B}_$rep.json 2> /dev/null; echo "rc=$?" >> $O/rc.txt
 done
done

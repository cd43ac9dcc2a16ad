#!/bin/bash
# One gpurun call: GPU tests, smoke, and every bench.py mode. Usage (on the box, from the repo root):
#   bash tools/gpu_check.sh <outdir> [pytest-args...]
set -u
OUT=${1:-gpurun_out/check}; shift || true
mkdir -p "$OUT"
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG" > "$OUT/info.txt"
timeout 1200 python -m pytest tests -m gpu -x -q "$@" > "$OUT/pytest.log" 2>&1; echo "pytest_rc=$?" >> "$OUT/pytest.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke_rc=$?" >> "$OUT/smoke.log"
timeout 400 python bench.py --gpus 1 --steps 20 --warmup 5 > "$OUT/bench1.json" 2> "$OUT/bench1.err"
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2960$N bench.py --gpus $N --steps 20 --warmup 5 > "$OUT/bench$N.json" 2> "$OUT/bench$N.err"
  timeout 400 python bench.py --gpus $N --steps 20 --warmup 5 > "$OUT/bench${N}_sp.json" 2> "$OUT/bench${N}_sp.err"
done
[ "$NG" -ge 4 ] && timeout 400 python bench.py --gpus 4 --ranks 8 --steps 20 --warmup 5 > "$OUT/bench4_r8_sp.json" 2> "$OUT/bench4_r8_sp.err"
true

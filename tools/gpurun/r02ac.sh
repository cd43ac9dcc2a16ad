O=gpurun_out/r02ac; mkdir -p $O
for M in 0 1; do for rep in 1 2; do
PAT_GROUP_LOCAL=$M timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $O/b1_m${M}_$rep.json 2> $O/b1_m${M}_$rep.err
done; done
timeout 600 python -m pytest tests/test_gpu_group.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log

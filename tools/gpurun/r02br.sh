O=gpurun_out/r02br; mkdir -p $O
for rep in 1 2 3; do for V in "" early; do
PAT_LIB_VARIANT=$V timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $O/b1_${V:-base}_$rep.json 2> $O/b1_${V:-base}_$rep.err
done; done

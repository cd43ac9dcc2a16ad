set -u
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/rc.txt
for i in 1 2; do timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench1_$i.json 2> $O/bench1_$i.err; echo "rc_b1_$i=$?" >> $O/rc.txt; done
timeout 200 python tools/eager_probe.py > $O/eager_probe.json 2> $O/eager_probe.err

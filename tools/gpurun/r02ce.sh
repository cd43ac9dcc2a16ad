# final N=1 bench line (default command) after the e2e set-count rule, and its reference arm
set -u
O=gpurun_out/r02ce; mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "rc_b1=$?" >> $O/rc.txt
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref1.json 2> $O/ref1.err; echo "rc_ref1=$?" >> $O/rc.txt

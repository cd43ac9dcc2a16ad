"""Print a PAT vs NCCL table from bench_sweep.py output files."""
import json
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    print("==", f)
    t = defaultdict(dict)
    for line in open(f):
        r = json.loads(line)
        t[(r["coll"], r["dtype"], r["bytes_per_rank"])][r["impl"]] = r
    for k in sorted(t):
        d = t[k]
        p = d.get("pat") or next(v for kk, v in d.items() if kk.startswith("pat"))
        nc = next((v for kk, v in d.items() if kk.startswith("nccl")), None)
        s = f"{k[0]} {k[1]:4s} {k[2]:>11d} pat {p['us']:8.1f}us {p['busbw_gbs']:6.1f}GB/s"
        if "plan" in p:
            s += f" P{p['plan']['protocol']} ch{p['plan']['channels']:<3d} it{p['plan']['iterations']:<4d}"
        if nc:
            s += f" | nccl {nc['us']:8.1f}us {nc['busbw_gbs']:6.1f}  x{nc['us'] / p['us']:.2f}"
        print(s)

"""CPU checks that the headline numbers quoted in DESIGN.md follow from the committed evidence
under profiles/ (the ncu NVLink captures and the graph-mode sweeps against NCCL Ring)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def test_nvlink_capture_summary():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_nvlink.py"),
                          os.path.join(P, "r01f_ncu_nvlink_g2.csv"), "--log", os.path.join(P, "r01f_ncu_nvlink_g2.log")],
                         capture_output=True, text=True, check=True).stdout
    rows = [l for l in out.splitlines() if l.startswith("ag 256 MiB n=2 proto 2") and "warm-up" not in l]
    assert rows, out
    f = rows[0].split()
    egress_user, egress_wire, ratio = float(f[-3]), float(f[-2]), float(f[-1])
    assert 600 < egress_user < 720 and 740 < egress_wire < 800 and abs(ratio - 1.191) < 0.01


def test_pat_beats_nccl_ring_at_every_size_to_1mib():
    for n in (2, 3, 4):
        d = {}
        for line in open(os.path.join(P, f"r01f_sweep_n{n}_graph.jsonl")):
            r = json.loads(line)
            d[(r["coll"], r["impl"], r["bytes_per_rank"])] = r["us"]
        sizes = sorted({k[2] for k in d if k[2] <= 1 << 20})
        assert len(sizes) >= 18
        for coll in ("ag", "rs"):
            for b in sizes:
                assert d[(coll, "pat", b)] * 2.0 < d[(coll, "nccl-Ring", b)], (n, coll, b)

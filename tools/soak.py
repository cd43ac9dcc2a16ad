"""Soak test: random calls (sizes, dtypes, ops, protocols, placements, T) on long-lived
communicators for a fixed wall time, every result checked against the oracle. Catches rare
ordering races that short parity tests can miss.

  python tools/soak.py --seconds 300
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, mismatch, oracle_ag, oracle_rs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=7)
    args = ap.parse_args()
    ngpu = torch.cuda.device_count()
    rng = np.random.default_rng(args.seed)
    comms = {}
    calls = bad = 0
    t0 = time.time()
    while time.time() - t0 < args.seconds:
        n = int(rng.choice([2, 3, 4, 6, 8]))
        spread = ngpu >= 2 and rng.random() < 0.6
        devices = tuple(r % ngpu for r in range(n)) if spread else (0,) * n
        proto = int(rng.choice([0, 0, _lib.PROTO_LL, _lib.PROTO_SIMPLE, _lib.PROTO_PULL]))
        key = (devices, proto)
        if key not in comms:
            if len(comms) >= 6:
                k, c = comms.popitem()
                c.destroy()
            comms[key] = PatComm.init_all(n, list(devices), protocol=proto, channels=int(rng.choice([4, 16, 64])),
                                          staging_bytes=n * 1024 * 1024, fused=-1)
        comm = comms[key]
        dt = int(rng.choice([O.INT32, O.FLOAT32, O.BFLOAT16, O.FLOAT16, O.INT8, O.FLOAT64]))
        elems = int(rng.integers(1, 300000))
        p = O.random_payload(dt, n, elems, calls)
        got = gpu_allgather(comm, list(devices), p, elems, dt)
        want = oracle_ag(n, O.max_trees(n), dt, p, elems)
        m = mismatch(got, want, elems)
        if m:
            bad += 1
            print("AG", n, devices, proto, dt, elems, m, flush=True)
        op = int(rng.choice([O.SUM, O.MAX]))
        q = O.random_payload(dt, n * n, elems, calls + 7)
        got = gpu_reduce_scatter(comm, list(devices), q, elems, dt, op)
        want = oracle_rs(n, O.max_trees(n), dt, op, q, elems)
        m = mismatch(got, want, elems)
        if m:
            bad += 1
            print("RS", n, devices, proto, dt, op, elems, m, flush=True)
        calls += 2
    for c in comms.values():
        assert c.async_error() == 0
        c.destroy()
    print(f"soak: {calls} calls in {time.time() - t0:.0f} s, {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

"""LL128 mismatch intervals (debug tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from test_gpu_parity import gpu_allgather, oracle_ag  # noqa: E402

n = 4
devices = [0] * n
for chan, stag in ((8, n * 256 * 1024), (1, n * 256 * 1024), (8, 0)):
    comm = PatComm.init_all(n, devices, protocol=_lib.PROTO_LL128, staging_bytes=stag, channels=chan, fused=-1)
    print("plan", comm.plan(0, 70001, O.BFLOAT16), flush=True)
    for dt, elems in ((O.BFLOAT16, 70001), (O.UINT8, 140002), (O.FLOAT32, 35001), (O.FLOAT16, 70001), (O.BFLOAT16, 70000), (O.INT8, 140001)):
        p = O.random_payload(dt, n, elems, 7)
        got = gpu_allgather(comm, devices, p, elems, dt)
        want = oracle_ag(n, O.max_trees(n), dt, p, elems)
        es = p.itemsize
        for r in range(n):
            g, w = got[r].view(np.uint8), want[r].view(np.uint8)
            d = np.nonzero(g != w)[0]
            if d.size:
                cb = elems * es
                # intervals
                iv, s0, prev = [], d[0], d[0]
                for x in d[1:]:
                    if x != prev + 1:
                        iv.append((s0, prev)); s0 = x
                    prev = x
                iv.append((s0, prev))
                print(f"chan={chan} dt={dt} elems={elems} rank={r}: {d.size} bad bytes; intervals (origin, off0, off1):",
                      [(int(a // cb), int(a % cb), int(b % cb)) for a, b in iv[:12]], flush=True)
                # what values: got vs want at the first bad position
                a = d[0]
                print("   got", g[a:a + 16].tolist(), "want", w[a:a + 16].tolist(), flush=True)
    comm.destroy()

"""Stress the polling protocols (LL, LL32) against the oracle on odd sizes and 2-byte elements;
print where mismatches are (debug tool). ITERS (env) sets the repetitions per configuration."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, oracle_ag, oracle_rs  # noqa: E402

ngpu = torch.cuda.device_count()
for n, devices in ((8, [r % ngpu for r in range(8)]), (8, [0] * 8), (4, list(range(min(4, ngpu))) if ngpu >= 4 else [0] * 4)):
    for proto in (_lib.PROTO_LL, _lib.PROTO_LL32):
        comm = PatComm.init_all(n, devices, protocol=proto, staging_bytes=n * 256 * 1024, channels=8, fused=-1)
        bad = 0
        for it in range(int(os.environ.get("ITERS", "6"))):
            for elems in (70001, 4099, 65536, 123457, 1000003):
                for dt in (O.BFLOAT16, O.FLOAT32, O.INT32):
                    q = O.random_payload(dt, n * n, elems, elems + it)
                    got = gpu_reduce_scatter(comm, devices, q, elems, dt, O.SUM)
                    want = oracle_rs(n, O.max_trees(n), dt, O.SUM, q, elems)
                    for r in range(n):
                        g, w = got[r].view(np.uint8), want[r].view(np.uint8)
                        if not np.array_equal(g, w):
                            d = np.nonzero(g != w)[0]
                            bad += 1
                            print(f"RS n={n} dev={devices} proto={proto} it={it} elems={elems} dt={dt} rank={r}: "
                                  f"{d.size} bytes differ, first {d[:8]} last {d[-4:]}", flush=True)
                    p = O.random_payload(dt, n, elems, elems + it + 100)
                    got = gpu_allgather(comm, devices, p, elems, dt)
                    want = oracle_ag(n, O.max_trees(n), dt, p, elems)
                    for r in range(n):
                        g, w = got[r].view(np.uint8), want[r].view(np.uint8)
                        if not np.array_equal(g, w):
                            d = np.nonzero(g != w)[0]
                            bad += 1
                            print(f"AG n={n} dev={devices} proto={proto} it={it} elems={elems} dt={dt} rank={r}: "
                                  f"{d.size} bytes differ, first {d[:8]}", flush=True)
        print(f"n={n} devices={devices} proto={proto}: {bad} bad", flush=True)
        comm.destroy()

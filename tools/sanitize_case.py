"""Small AG/RS cases for compute-sanitizer (memcheck): fused executor, and the transport kernel
with every protocol, 4 logical ranks on cuda:0, checked against the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, oracle_ag, oracle_rs  # noqa: E402

n = 4
bad = 0
for fused, proto in ((0, 0), (-1, _lib.PROTO_LL), (-1, _lib.PROTO_SIMPLE), (-1, _lib.PROTO_PULL)):
    comm = PatComm.init_all(n, [0] * n, fused=fused, protocol=proto, channels=2, staging_bytes=n * 64 * 1024)
    for elems in (1, 777, 5000):
        p = O.random_payload(O.BFLOAT16, n, elems, elems)
        got = gpu_allgather(comm, [0] * n, p, elems, O.BFLOAT16)
        want = oracle_ag(n, O.max_trees(n), O.BFLOAT16, p, elems)
        bad += sum(not np.array_equal(got[r], want[r]) for r in range(n))
        q = O.random_payload(O.FLOAT32, n * n, elems, elems + 1)
        got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT32, O.SUM)
        want = oracle_rs(n, O.max_trees(n), O.FLOAT32, O.SUM, q, elems)
        bad += sum(not np.array_equal(got[r], want[r]) for r in range(n))
    comm.destroy()
print(f"sanitize_case: {bad} mismatches")
sys.exit(1 if bad else 0)

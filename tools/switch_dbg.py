"""Protocol-switch sequence of test_protocol_switches_share_no_inbox_state with mismatch details."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm  # noqa: E402
from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, oracle_ag, oracle_rs  # noqa: E402

n = 4
for variant in ("full", "no-bulk", "no-rs"):
    comm = PatComm.init_all(n, [0] * n, fused=-1, channels=2, staging_bytes=n * 32 * 1024, ll_threshold=16384)
    for it in range(16):
        elems = [200, 5000, 60000, 3000][it % 4]
        if variant == "no-bulk" and elems == 60000:
            continue
        p = (np.arange(n * elems, dtype=np.int64) % 64 + 1 + it).astype(np.int32)
        got = gpu_allgather(comm, [0] * n, p, elems, O.INT32)
        want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
        for r in range(n):
            d = np.nonzero(got[r] != want[r])[0]
            if d.size:
                print(f"{variant} AG it={it} elems={elems} plan={comm.plan(0, elems, O.INT32)} rank={r}: {d.size} elems bad, "
                      f"first {(d[:6] // elems).tolist()} {(d[:6] % elems).tolist()} got {got[r][d[:6]].tolist()} "
                      f"want {want[r][d[:6]].tolist()}", flush=True)
        if variant == "no-rs":
            continue
        q = (np.arange(n * n * elems, dtype=np.int64) % 64 + it).astype(np.int32)
        got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.INT32, O.SUM)
        want = oracle_rs(n, O.max_trees(n), O.INT32, O.SUM, q, elems)
        for r in range(n):
            d = np.nonzero(got[r] != want[r])[0]
            if d.size:
                print(f"{variant} RS it={it} elems={elems} rank={r}: {d.size} bad, first {d[:6].tolist()}", flush=True)
    print(variant, "done", flush=True)
    comm.destroy()

"""Long protocol-switching sequence on one communicator (LL / SIMPLE / PULL by size),
AG and RS interleaved, buffers re-allocated every call; counts mismatches (debug tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, mismatch, oracle_ag, oracle_rs  # noqa: E402

ngpu = torch.cuda.device_count()
rng = np.random.default_rng(1)
for n, devices in ((4, [0] * 4), (4, list(range(4)) if ngpu >= 4 else [0] * 4), (8, [r % ngpu for r in range(8)])):
    for forced in (0, _lib.PROTO_PULL):
        comm = PatComm.init_all(n, devices, fused=-1, channels=2, staging_bytes=n * 32 * 1024, ll_threshold=16384,
                                protocol=forced)
        bad = 0
        for it in range(60):
            elems = int(rng.choice([200, 3000, 5000, 60000, 100003]))
            p = (np.arange(n * elems, dtype=np.int64) % 64 + 1 + it).astype(np.int32)
            got = gpu_allgather(comm, devices, p, elems, O.INT32)
            want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
            m = mismatch(got, want, elems)
            if m:
                bad += 1
                print(f"n={n} dev={devices} forced={forced} AG it={it} elems={elems} "
                      f"proto={comm.plan(0, elems, O.INT32)['protocol']}: {m}", flush=True)
            q = (np.arange(n * n * elems, dtype=np.int64) % 64 + it).astype(np.int32)
            got = gpu_reduce_scatter(comm, devices, q, elems, O.INT32, O.SUM)
            want = oracle_rs(n, O.max_trees(n), O.INT32, O.SUM, q, elems)
            m = mismatch(got, want, elems)
            if m:
                bad += 1
                print(f"n={n} dev={devices} forced={forced} RS it={it} elems={elems} "
                      f"proto={comm.plan(1, elems, O.INT32)['protocol']}: {m}", flush=True)
        print(f"n={n} devices={devices} forced={forced}: {bad} bad", flush=True)
        comm.destroy()

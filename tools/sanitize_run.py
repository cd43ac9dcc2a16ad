"""Small transport suite for compute-sanitizer (memcheck / racecheck / synccheck, ONE tool per
gpurun call): n = 4 logical ranks on cuda:0 through the transport kernel (fused = -1), every
protocol (LL, LL32, SIMPLE, PULL), all-gather and reduce-scatter (fp32 sum, bf16 sum), sizes that
take the vector, tail and multi-step paths; results checked bit-exact against the CPU oracle.
Exit 0 only if every result matches.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PAT_TIMEOUT_MS", "300000")  # instrumented kernels run far slower

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm  # noqa: E402

PROTOS = {"LL": 1, "SIMPLE": 2, "PULL": 3, "LL32": 5}


def run(comm, n, dt, elems, seed):
    dev = "cuda:0"
    p = O.random_payload(dt, n, elems, seed)
    es = p.itemsize
    s = [torch.from_numpy(p[r * elems:(r + 1) * elems].copy().view(np.uint8)).to(dev) for r in range(n)]
    r_ = [torch.zeros(n * elems * es, dtype=torch.uint8, device=dev) for _ in range(n)]
    comm.all_gather(s, r_, elems, dt)
    torch.cuda.synchronize()
    want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
    bad = sum(r_[r].cpu().numpy().tobytes() != want[r].tobytes() for r in range(n))
    q = O.random_payload(dt, n * n, elems, seed + 1)
    s = [torch.from_numpy(q[r * n * elems:(r + 1) * n * elems].copy().view(np.uint8)).to(dev) for r in range(n)]
    r_ = [torch.zeros(elems * es, dtype=torch.uint8, device=dev) for _ in range(n)]
    comm.reduce_scatter(s, r_, elems, dt, O.SUM)
    torch.cuda.synchronize()
    want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
    bad += sum(r_[r].cpu().numpy().tobytes() != want[r].tobytes() for r in range(n))
    comm.raise_async_error()
    return bad


def main():
    n = 4
    fails = 0
    for name, proto in PROTOS.items():
        # small slots so the mid size runs several pipeline steps per channel
        comm = PatComm.init_all(n, [0] * n, fused=-1, protocol=proto, channels=4, slice_bytes=64 << 10)
        for dt in (O.FLOAT32, O.BFLOAT16):
            for elems in (1, 37, 4099, 100_003):
                b = run(comm, n, dt, elems, 7 * elems + dt)
                print(f"{name} dt={dt} elems={elems} bad_ranks={b}", flush=True)
                fails += b
        comm.destroy()
    print(f"SANITIZE_SUITE fails={fails}", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

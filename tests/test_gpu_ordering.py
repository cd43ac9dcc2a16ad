"""Calls of one communicator issued on different streams, with no synchronisation between the
streams, still run one after the other on each device (NCCL's guarantee): transport calls share
the channels' flags, step counters and inbox slots. Bit-exact against the CPU oracle."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PatComm  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("n,spread", [(4, False), (4, True), (2, True)])  # (2, True): one rank per GPU,
@pytest.mark.parametrize("elems", [3000, 262144, 1 << 20])  # LL, LL32, SIMPLE   non-cooperative launches
def test_calls_on_two_streams(n, spread, elems):
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    devices = [r % NGPU for r in range(n)] if spread else [0] * n
    comm = PatComm.init_all(n, devices, fused=-1)
    try:
        dset = sorted(set(devices))
        sa = {d: torch.cuda.Stream(d) for d in dset}
        sb = {d: torch.cuda.Stream(d) for d in dset}
        jobs = []
        for it in range(12):
            p = O.random_payload(O.FLOAT32, n, elems, 100 * it + 1)
            q = O.random_payload(O.FLOAT32, n * n, elems, 100 * it + 2)
            ag_s = [torch.from_numpy(p[r * elems:(r + 1) * elems].copy()).to(f"cuda:{devices[r]}") for r in range(n)]
            ag_r = [torch.zeros(n * elems, device=f"cuda:{devices[r]}") for r in range(n)]
            rs_s = [torch.from_numpy(q[r * n * elems:(r + 1) * n * elems].copy()).to(f"cuda:{devices[r]}")
                    for r in range(n)]
            rs_r = [torch.zeros(elems, device=f"cuda:{devices[r]}") for r in range(n)]
            jobs.append((p, q, ag_r, rs_r, ag_s, rs_s))
        for d in dset:
            torch.cuda.synchronize(d)
        # all-gathers on stream A, reduce-scatters on stream B: unordered, A's and B's kernels would
        # run at the same time (small calls' CTAs are co-resident) on the same channels
        for p, q, ag_r, rs_r, ag_s, rs_s in jobs:
            comm.all_gather(ag_s, ag_r, elems, O.FLOAT32, streams=[sa[d] for d in devices])
            comm.reduce_scatter(rs_s, rs_r, elems, O.FLOAT32, O.SUM, streams=[sb[d] for d in devices])
        for d in dset:
            torch.cuda.synchronize(d)
        comm.raise_async_error()
        for p, q, ag_r, rs_r, _, _ in jobs:
            want_ag, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), O.FLOAT32, p, elems)
            want_rs, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.FLOAT32, O.SUM, q, elems)
            for r in range(n):
                assert ag_r[r].cpu().numpy().tobytes() == want_ag[r].tobytes(), ("AG", r)
                assert rs_r[r].cpu().numpy().tobytes() == want_rs[r].tobytes(), ("RS", r)
    finally:
        comm.destroy()

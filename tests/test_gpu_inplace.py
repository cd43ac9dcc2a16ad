"""In-place collectives, as NCCL allows them: an all-gather whose send buffer is the rank's own slot
of its receive buffer (sendbuf == recvbuf + rank * count), and a reduce-scatter whose receive
buffer is the rank's own block of its send buffer (recvbuf == sendbuf + rank * count) — the form
FSDP / ZeRO-3 callers use. Bit-exact against the CPU oracle for every executor and protocol."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PatComm  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
CASES = [(4, False, 0, 0), (4, False, -1, 0), (2, True, 0, 0), (4, True, 0, 0), (4, False, -1, 3), (4, True, 0, 3),
         (4, True, 0, 2)]  # (n, spread, fused, protocol: 0 auto, 3 PULL, 2 SIMPLE)


@pytest.mark.parametrize("n,spread,fused,proto", CASES)
@pytest.mark.parametrize("elems", [1, 3000, 262144, 1 << 21])
def test_inplace(n, spread, fused, proto, elems):
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    devices = [r % NGPU for r in range(n)] if spread else [0] * n
    comm = PatComm.init_all(n, devices, fused=fused, protocol=proto)
    dt = O.FLOAT32
    try:
        p = O.random_payload(dt, n, elems, 7 * elems + n)
        bufs = []
        for r in range(n):
            b = torch.zeros(n * elems, dtype=torch.float32, device=f"cuda:{devices[r]}")
            b[r * elems:(r + 1) * elems] = torch.from_numpy(p[r * elems:(r + 1) * elems].copy())
            bufs.append(b)
        comm.all_gather([b[r * elems:(r + 1) * elems] for r, b in enumerate(bufs)], bufs, elems, dt)
        for d in sorted(set(devices)):
            torch.cuda.synchronize(d)
        want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
        for r in range(n):
            assert bufs[r].cpu().numpy().tobytes() == want[r].tobytes(), ("AG", r)
        q = O.random_payload(dt, n * n, elems, 11 * elems + n)
        bufs = [torch.from_numpy(q[r * n * elems:(r + 1) * n * elems].copy()).to(f"cuda:{devices[r]}")
                for r in range(n)]
        comm.reduce_scatter(bufs, [b[r * elems:(r + 1) * elems] for r, b in enumerate(bufs)], elems, dt, O.SUM)
        for d in sorted(set(devices)):
            torch.cuda.synchronize(d)
        want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
        for r in range(n):
            got = bufs[r].cpu().numpy()[r * elems:(r + 1) * elems]
            assert np.ascontiguousarray(got).tobytes() == want[r].tobytes(), ("RS", r)
        comm.raise_async_error()
    finally:
        comm.destroy()

"""Device-side statistics against the reference: the intermediate-slot occupancy per round, counted
by the transport kernel while it runs (PAT_STATS=1, patCommStatsRead), equals the reference
executor's ExecStats.occupancy_per_round (StatsBuilder::add_round, simulate.cpp:109-129; the
brute-force trackers of tests/brute_force.hpp:25-54) for every rank count 2..8 and every valid T,
all-gather and reduce-scatter. The expected values are the reference's own (tests/golden/executor.npz).
Also: the device barrier (patCommBarrier) across GPUs."""
import os

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PROTO_SIMPLE, SUM, FLOAT32, PatComm  # noqa: E402
from paper_2506_20252_b200 import schedule as S  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(comm, devices, n, kind, sched, elems=4096):
    sb, rb = [], []
    for r in range(n):
        d = f"cuda:{devices[r]}"
        if kind == "ag":
            sb.append(torch.rand(elems, device=d))
            rb.append(torch.empty(n * elems, device=d))
        else:
            sb.append(torch.rand(n * elems, device=d))
            rb.append(torch.empty(elems, device=d))
    if kind == "ag":
        comm.all_gather(sb, rb, elems, FLOAT32, schedule=sched)
    else:
        comm.reduce_scatter(sb, rb, elems, FLOAT32, SUM, schedule=sched)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    comm.raise_async_error()
    return comm.device_occupancy()


@pytest.mark.parametrize("spread", [False, True])
def test_device_occupancy_equals_reference(golden_dir, monkeypatch, spread):
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    monkeypatch.setenv("PAT_STATS", "1")
    ex = np.load(os.path.join(golden_dir, "executor.npz"))
    checked = 0
    for n in range(2, 9):
        devices = [r % NGPU for r in range(n)] if spread else [0] * n
        comm = PatComm.init_all(n, devices, fused=-1, protocol=PROTO_SIMPLE)
        try:
            for t in O.valid_tree_counts(n):
                key = f"n{n}_t{t}_s0_d4"
                want_ag = [int(x) for x in ex[f"ag_stats_{key}"][6:]]
                want_rs = [int(x) for x in ex[f"rs_stats_{key}"][6:]]
                got = _run(comm, devices, n, "ag", S.pat_allgather(n, t))
                assert got == [want_ag] * n, (n, t, "ag", got, want_ag)
                got = _run(comm, devices, n, "rs", S.pat_reduce_scatter(n, t))
                assert got == [want_rs] * n, (n, t, "rs", got, want_rs)
                checked += 2
        finally:
            comm.destroy()
    assert checked == 2 * sum(len(O.valid_tree_counts(n)) for n in range(2, 9))


def test_device_barrier_orders_ranks():
    """patCommBarrier: rank 1's stream is held back by a spin; after the barrier, rank 0's stream
    cannot run ahead of rank 1's spin (checked through the elapsed time on rank 0's stream)."""
    if NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    comm = PatComm.init_all(2, [0, 1])
    try:
        s = [torch.cuda.Stream(0), torch.cuda.Stream(1)]
        for _ in range(3):
            comm.barrier(s)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(0), torch.cuda.stream(s[0]):
            e0.record(s[0])
        with torch.cuda.device(1), torch.cuda.stream(s[1]):
            torch.cuda._sleep(20_000_000)  # ~10 ms on rank 1 only
        comm.barrier(s)
        with torch.cuda.device(0), torch.cuda.stream(s[0]):
            e1.record(s[0])
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        comm.raise_async_error()
        assert e0.elapsed_time(e1) > 5.0  # ms: rank 0 waited for rank 1
    finally:
        comm.destroy()

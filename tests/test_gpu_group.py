"""Grouped collectives (patGroupStart / patGroupEnd): an all-gather and a reduce-scatter (sum) of one
communicator become one launch — the fused single-device kernel, or the transport kernel with each
call on half of the channels — and must give exactly the results of the two calls made alone
(bit-exact against the CPU oracle), in any order, interleaved with ungrouped calls."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PatComm, group  # noqa: E402
from paper_2506_20252_b200 import _lib  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _bufs(devices, dt, n, elems, seed, pad=0):
    """Device buffers for one AG and one RS call, and the oracle's expected outputs."""
    p = O.random_payload(dt, n, elems, seed)
    q = O.random_payload(dt, n * n, elems, seed + 1)
    es = p.itemsize
    mk = lambda a, d: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(f"cuda:{d}")  # noqa: E731
    ag_s = [mk(p[r * elems:(r + 1) * elems], devices[r]) for r in range(n)]
    ag_r = [torch.zeros(n * elems * es + pad, dtype=torch.uint8, device=f"cuda:{devices[r]}") for r in range(n)]
    rs_s = [mk(q[r * n * elems:(r + 1) * n * elems], devices[r]) for r in range(n)]
    rs_r = [torch.zeros(elems * es + pad, dtype=torch.uint8, device=f"cuda:{devices[r]}") for r in range(n)]
    want_ag, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
    want_rs, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
    ptr = lambda t: t.data_ptr() + pad  # noqa: E731
    return dict(ag_s=ag_s, ag_r=ag_r, rs_s=rs_s, rs_r=rs_r, want_ag=want_ag, want_rs=want_rs, es=es,
                ag_sp=[t.data_ptr() for t in ag_s], ag_rp=[ptr(t) for t in ag_r],
                rs_sp=[t.data_ptr() for t in rs_s], rs_rp=[ptr(t) for t in rs_r], pad=pad)


def _check(b, devices, n, elems, tag):
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    pad, es = b["pad"], b["es"]
    for r in range(n):
        got = b["ag_r"][r].cpu().numpy()[pad:pad + n * elems * es]
        assert got.tobytes() == b["want_ag"][r].tobytes(), (tag, "AG", r)
        got = b["rs_r"][r].cpu().numpy()[pad:pad + elems * es]
        assert got.tobytes() == b["want_rs"][r].tobytes(), (tag, "RS", r)


def _grouped(comm, b, elems, dt, rs_first=False):
    with group():
        if rs_first:
            comm.reduce_scatter(b["rs_sp"], b["rs_rp"], elems, dt, O.SUM)
            comm.all_gather(b["ag_sp"], b["ag_rp"], elems, dt)
        else:
            comm.all_gather(b["ag_sp"], b["ag_rp"], elems, dt)
            comm.reduce_scatter(b["rs_sp"], b["rs_rp"], elems, dt, O.SUM)


@pytest.mark.parametrize("dt", [O.FLOAT32, O.BFLOAT16, O.INT32, O.FLOAT64])
@pytest.mark.parametrize("elems,pad", [(8192, 0), (262144, 0), (1000, 0), (4097, 0), (8192, 16)])
def test_group_fused_single_device(dt, elems, pad):
    """8 ranks on one GPU: the fused group kernel (32-byte aligned) or the one-by-one fallback."""
    n = 8
    comm = PatComm.init_all(n, [0] * n)
    try:
        for rs_first in (False, True):
            b = _bufs([0] * n, dt, n, elems, 11 * elems + dt + rs_first, pad)
            _grouped(comm, b, elems, dt, rs_first)
            _check(b, [0] * n, n, elems, ("fused", rs_first))
        comm.raise_async_error()
    finally:
        comm.destroy()


@pytest.mark.parametrize("spread", [False, True])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_group_transport(spread, n):
    """The transport group kernel: LL, LL32 and SIMPLE sizes, both orders, then ungrouped calls on
    the same communicator (whose channels the grouped reduce-scatter's half does not share)."""
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    devices = [r % NGPU for r in range(n)] if spread else [0] * n
    comm = PatComm.init_all(n, devices, fused=-1)
    try:
        for it, elems in enumerate((64, 3000, 262144, 1 << 21)):  # LL, LL, LL32, SIMPLE/LL32 by n
            dt = (O.FLOAT32, O.BFLOAT16, O.INT32, O.FLOAT32)[it]
            for rs_first in (False, True):
                b = _bufs(devices, dt, n, elems, 7 * elems + it + rs_first)
                _grouped(comm, b, elems, dt, rs_first)
                _check(b, devices, n, elems, ("group", elems, rs_first))
            b = _bufs(devices, dt, n, elems, 5 * elems + it)
            comm.all_gather(b["ag_sp"], b["ag_rp"], elems, dt)
            comm.reduce_scatter(b["rs_sp"], b["rs_rp"], elems, dt, O.SUM)
            _check(b, devices, n, elems, ("alone", elems))
        comm.raise_async_error()
    finally:
        comm.destroy()


def test_group_three_calls_and_non_sum():
    """AG, RS, AG in one group (a pair + a single); a max reduce-scatter is launched on its own."""
    n = 4
    devices = [r % max(NGPU, 1) for r in range(n)]
    comm = PatComm.init_all(n, devices, fused=-1)
    try:
        b1 = _bufs(devices, O.FLOAT32, n, 5000, 1)
        b2 = _bufs(devices, O.FLOAT32, n, 7000, 2)
        with group():
            comm.all_gather(b1["ag_sp"], b1["ag_rp"], 5000, O.FLOAT32)
            comm.reduce_scatter(b1["rs_sp"], b1["rs_rp"], 5000, O.FLOAT32, O.SUM)
            comm.all_gather(b2["ag_sp"], b2["ag_rp"], 7000, O.FLOAT32)
        for d in sorted(set(devices)):
            torch.cuda.synchronize(d)
        for r in range(n):
            assert b1["ag_r"][r].cpu().numpy().tobytes() == b1["want_ag"][r].tobytes()
            assert b1["rs_r"][r].cpu().numpy().tobytes() == b1["want_rs"][r].tobytes()
            assert b2["ag_r"][r].cpu().numpy().tobytes() == b2["want_ag"][r].tobytes()
        p = O.random_payload(O.INT32, n * n, 3000, 9)
        s = [torch.from_numpy(p[r * n * 3000:(r + 1) * n * 3000].copy()).to(f"cuda:{devices[r]}") for r in range(n)]
        rr = [torch.zeros(3000, dtype=torch.int32, device=f"cuda:{devices[r]}") for r in range(n)]
        a = _bufs(devices, O.INT32, n, 3000, 10)
        with group():
            comm.all_gather(a["ag_sp"], a["ag_rp"], 3000, O.INT32)
            comm.reduce_scatter(s, rr, 3000, O.INT32, O.MAX)
        for d in sorted(set(devices)):
            torch.cuda.synchronize(d)
        want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.INT32, O.MAX, p, 3000)
        for r in range(n):
            assert rr[r].cpu().numpy().tobytes() == want[r].tobytes()
            assert a["ag_r"][r].cpu().numpy().tobytes() == a["want_ag"][r].tobytes()
        comm.raise_async_error()
    finally:
        comm.destroy()


def test_group_graph_capture():
    """A grouped pair captured into a CUDA graph and replayed."""
    n = 4
    devices = [r % max(NGPU, 1) for r in range(n)]
    comm = PatComm.init_all(n, devices, fused=-1)
    try:
        b = _bufs(devices, O.FLOAT32, n, 65536, 3)
        streams = {d: torch.cuda.Stream(d) for d in sorted(set(devices))}
        st = [streams[d] for d in devices]
        _grouped(comm, b, 65536, O.FLOAT32)  # warm: pools, compiled plans
        for d in streams:
            torch.cuda.synchronize(d)
        graphs = {d: torch.cuda.CUDAGraph() for d in streams}
        for d in streams:
            streams[d].wait_stream(torch.cuda.current_stream(d))
            with torch.cuda.device(d):
                torch.cuda.set_stream(streams[d])
                graphs[d].capture_begin(capture_error_mode="relaxed")
        with group():
            comm.all_gather(b["ag_sp"], b["ag_rp"], 65536, O.FLOAT32, streams=st)
            comm.reduce_scatter(b["rs_sp"], b["rs_rp"], 65536, O.FLOAT32, O.SUM, streams=st)
        for d in streams:
            with torch.cuda.device(d):
                graphs[d].capture_end()
                torch.cuda.set_stream(torch.cuda.default_stream(d))
        for r in range(n):
            b["ag_r"][r].zero_()
            b["rs_r"][r].zero_()
        for d in streams:
            torch.cuda.synchronize(d)
        for _ in range(3):
            for d in streams:
                with torch.cuda.device(d):
                    graphs[d].replay()
        _check(b, devices, n, 65536, "graph")
        comm.raise_async_error()
    finally:
        comm.destroy()


@pytest.mark.parametrize("spread", [False, True])
@pytest.mark.parametrize("n", [2, 4])
def test_group_mixed_sizes(spread, n):
    """A pair whose halves take different protocols (an LL half spans fewer channels than an LL32
    or SIMPLE half): ranges that would share channels run one after the other, the rest as one
    launch; every combination bit-exact, then the fused single-device executor with unequal sizes."""
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    devices = [r % NGPU for r in range(n)] if spread else [0] * n
    comm = PatComm.init_all(n, devices, fused=-1)
    try:
        for ag_elems, rs_elems in ((262144, 64), (64, 262144), (1 << 21, 3000), (3000, 1 << 21), (64, 8)):
            for rs_first in (False, True):
                a = _bufs(devices, O.FLOAT32, n, ag_elems, 13 * ag_elems + rs_first)
                b = _bufs(devices, O.FLOAT32, n, rs_elems, 17 * rs_elems + rs_first + 1)
                with group():
                    if rs_first:
                        comm.reduce_scatter(b["rs_sp"], b["rs_rp"], rs_elems, O.FLOAT32, O.SUM)
                        comm.all_gather(a["ag_sp"], a["ag_rp"], ag_elems, O.FLOAT32)
                    else:
                        comm.all_gather(a["ag_sp"], a["ag_rp"], ag_elems, O.FLOAT32)
                        comm.reduce_scatter(b["rs_sp"], b["rs_rp"], rs_elems, O.FLOAT32, O.SUM)
                for d in sorted(set(devices)):
                    torch.cuda.synchronize(d)
                for r in range(n):
                    assert a["ag_r"][r].cpu().numpy().tobytes() == a["want_ag"][r].tobytes(), (ag_elems, rs_elems, r)
                    assert b["rs_r"][r].cpu().numpy().tobytes() == b["want_rs"][r].tobytes(), (ag_elems, rs_elems, r)
        comm.raise_async_error()
    finally:
        comm.destroy()
    comm = PatComm.init_all(8, [0] * 8)
    try:
        for ag_elems, rs_elems in ((8192, 1000), (1000, 65536)):
            a = _bufs([0] * 8, O.BFLOAT16, 8, ag_elems, ag_elems)
            b = _bufs([0] * 8, O.BFLOAT16, 8, rs_elems, rs_elems + 1)
            with group():
                comm.all_gather(a["ag_sp"], a["ag_rp"], ag_elems, O.BFLOAT16)
                comm.reduce_scatter(b["rs_sp"], b["rs_rp"], rs_elems, O.BFLOAT16, O.SUM)
            torch.cuda.synchronize(0)
            for r in range(8):
                assert a["ag_r"][r].cpu().numpy().tobytes() == a["want_ag"][r].tobytes(), ("fused", ag_elems, r)
                assert b["rs_r"][r].cpu().numpy().tobytes() == b["want_rs"][r].tobytes(), ("fused", rs_elems, r)
        comm.raise_async_error()
    finally:
        comm.destroy()

"""GPU parity: the sm_100a PAT kernels, called through the C ABI, against the CPU oracle and
against the reference's own outputs (tests/golden/executor.npz).

Bar: bit-exact everywhere (all-gather is a copy; reduce-scatter reproduces the reference's
PAT fold order with per-hop rounding in the wire dtype, so floats are bit-exact too).
Ranks that outnumber the GPUs run as logical ranks inside one cooperative kernel per GPU.
"""
import os

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PatComm, PatError, _lib  # noqa: E402
from paper_2506_20252_b200 import schedule as S  # noqa: E402
from paper_2506_20252_b200 import simulate as SIM  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
NP = {O.INT8: np.int8, O.UINT8: np.uint8, O.INT32: np.int32, O.UINT32: np.uint32, O.INT64: np.int64,
      O.UINT64: np.uint64, O.FLOAT16: np.uint16, O.BFLOAT16: np.uint16, O.FLOAT32: np.float32,
      O.FLOAT64: np.float64}

_COMMS = {}


def comm_for(n, devices=None, **cfg):
    """Cached communicators; at most a few stay alive (each holds n inbox pools in HBM)."""
    devices = tuple(devices if devices is not None else [0] * n)
    key = (n, devices, tuple(sorted(cfg.items())))
    if key not in _COMMS:
        while len(_COMMS) >= 4:
            old = next(iter(_COMMS))
            c = _COMMS.pop(old)
            assert c.async_error() == 0, old
            c.destroy()
        _COMMS[key] = PatComm.init_all(n, list(devices), **cfg)
    else:
        _COMMS[key] = _COMMS.pop(key)  # most recently used last
    return _COMMS[key]


def to_dev(a: np.ndarray, dev, pad_front=0):
    """Byte tensor on `dev` holding `a`, optionally starting `pad_front` bytes into the allocation."""
    raw = np.ascontiguousarray(a).view(np.uint8)
    t = torch.zeros(raw.size + pad_front + 64, dtype=torch.uint8, device=dev)
    t[pad_front:pad_front + raw.size] = torch.from_numpy(raw.copy()).to(dev)
    return t, t.data_ptr() + pad_front


def sync_all(devs):
    for d in sorted(set(devs)):
        torch.cuda.synchronize(d)


def gpu_allgather(comm, devices, payload, elems, dtype, pad=0, inplace=False, schedule=None):
    n = len(devices)
    es = payload.itemsize
    keep, sptr, rptr = [], [], []
    for r in range(n):
        chunk = payload[r * elems:(r + 1) * elems]
        if inplace:
            full = np.zeros(n * elems, payload.dtype)
            full[r * elems:(r + 1) * elems] = chunk
            t, p = to_dev(full, f"cuda:{devices[r]}", pad)
            keep.append(t)
            rptr.append(p)
            sptr.append(p + r * elems * es)
        else:
            ts, ps = to_dev(chunk, f"cuda:{devices[r]}", pad)
            tr, pr = to_dev(np.zeros(n * elems, payload.dtype), f"cuda:{devices[r]}", pad)
            keep += [ts, tr]
            sptr.append(ps)
            rptr.append(pr)
    comm.all_gather(sptr, rptr, elems, dtype, schedule=schedule)
    sync_all(devices)
    comm.raise_async_error()
    outs = []
    for r in range(n):
        t = keep[r] if inplace else keep[2 * r + 1]
        b = t.cpu().numpy()[pad:pad + n * elems * es]
        outs.append(b.view(payload.dtype))
    return outs


def gpu_reduce_scatter(comm, devices, payload, elems, dtype, op, pad=0, schedule=None):
    n = len(devices)
    es = payload.itemsize
    keep, sptr, rptr = [], [], []
    for r in range(n):
        ts, ps = to_dev(payload[r * n * elems:(r + 1) * n * elems], f"cuda:{devices[r]}", pad)
        tr, pr = to_dev(np.zeros(elems, payload.dtype), f"cuda:{devices[r]}", pad)
        keep += [ts, tr]
        sptr.append(ps)
        rptr.append(pr)
    comm.reduce_scatter(sptr, rptr, elems, dtype, op, schedule=schedule)
    sync_all(devices)
    comm.raise_async_error()
    return [keep[2 * r + 1].cpu().numpy()[pad:pad + elems * es].view(payload.dtype) for r in range(n)]


def mismatch(got, want, elems):
    """Where outputs differ: [(rank, first bad element, count, (block, offset) of the first)]."""
    out = []
    for r, (g, w) in enumerate(zip(got, want)):
        d = np.nonzero(g.view(np.uint8) != w.view(np.uint8))[0] // g.itemsize
        if d.size:
            out.append((r, int(d[0]), int(np.unique(d).size), divmod(int(d[0]), elems), g[d[:4]].tolist(),
                        w[d[:4]].tolist()))
    return out


def oracle_ag(n, trees, dtype, payload, elems):
    out, _ = O.run_allgather(O.pat_allgather(n, trees), dtype, payload, elems)
    return out


def oracle_rs(n, trees, dtype, op, payload, elems):
    out, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, trees), dtype, op, payload, elems)
    return out


def same(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


# ------------------------------------------------------------------ golden: the reference's own outputs

def test_reference_outputs_bit_exact_via_simulate_api(golden_dir):
    ex = np.load(os.path.join(golden_dir, "executor.npz"))
    for key in ex["index"]:
        n, t, seed, dt = (int(x[1:]) for x in str(key).split("_"))
        if seed != 0 or n > 8:
            continue
        elems = 4
        p = ex[f"ag_in_{key}"]
        res = SIM.run_allgather(S.pat_allgather(n, t), SIM.Payload(n, elems, [p[r * elems:(r + 1) * elems] for r in range(n)]))
        assert same(np.concatenate(res.outputs), ex[f"ag_out_{key}"]), key
        p = ex[f"rs_in_{key}"]
        op = SIM.ReduceOp.WrappingIntSum if dt == O.INT64 else SIM.ReduceOp.FloatSum
        res = SIM.run_reduce_scatter(S.pat_reduce_scatter(n, t),
                                     SIM.Payload(n, elems, [p[c * elems:(c + 1) * elems] for c in range(n * n)]), op)
        assert same(np.concatenate(res.outputs), ex[f"rs_out_{key}"]), key  # float64 bit-exact
        ref_stats = [int(x) for x in ex[f"rs_stats_{key}"][6:]]
        assert res.stats["occupancy_per_round"] == ref_stats


def test_simulate_api_errors():
    s = S.pat_allgather(4, 2)
    good = SIM.Payload(4, 2, [np.zeros(2, np.int64) for _ in range(4)])
    with pytest.raises(PatError) as ei:
        SIM.run_allgather(s, SIM.Payload(4, 2, good.chunks[:3]))
    assert ei.value.kind == "PayloadShapeError"
    with pytest.raises(PatError) as ei:
        SIM.run_allgather(S.pat_reduce_scatter(4, 2), good)
    assert ei.value.kind == "SimulationError"
    bad = S.pat_allgather(4, 2)
    bad.rounds[0].chunk_offsets = [3]
    with pytest.raises(PatError) as ei:
        SIM.run_allgather(bad, good)
    assert ei.value.kind == "InvalidScheduleError"
    rs = SIM.Payload(4, 2, [np.zeros(2, np.int64) for _ in range(16)])
    with pytest.raises(PatError) as ei:
        SIM.run_reduce_scatter(S.pat_reduce_scatter(4, 2), rs, SIM.ReduceOp.FloatSum)
    assert ei.value.kind == "UnsupportedOpError"


# ------------------------------------------------------------------ local mode (n logical ranks, one GPU)

EXECUTORS = {"fused": 0, "transport": -1}


@pytest.mark.parametrize("executor", EXECUTORS)
@pytest.mark.parametrize("n", range(1, 9))
@pytest.mark.parametrize("elems", [1, 3, 64, 1000, 40000])
def test_allgather_local_all_trees(n, elems, executor):
    for t in O.valid_tree_counts(n):
        comm = comm_for(n, trees=t, fused=EXECUTORS[executor])
        p = O.random_payload(O.FLOAT32, n, elems, n * 100 + t)
        got = gpu_allgather(comm, [0] * n, p, elems, O.FLOAT32)
        want = oracle_ag(n, t, O.FLOAT32, p, elems)
        for r in range(n):
            assert same(got[r], want[r]), (n, t, elems, r)


@pytest.mark.parametrize("dt", [O.FLOAT32, O.BFLOAT16, O.FLOAT16, O.INT32, O.INT64, O.FLOAT64, O.UINT8, O.INT8,
                                O.UINT32, O.UINT64])
@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("executor", EXECUTORS)
def test_reduce_scatter_local_dtypes(dt, n, executor):
    for elems in (1, 7, 300, 20000):
        for t in O.valid_tree_counts(n):
            comm = comm_for(n, trees=t, fused=EXECUTORS[executor])
            p = O.random_payload(dt, n * n, elems, 7 * n + t + elems)
            got = gpu_reduce_scatter(comm, [0] * n, p, elems, dt, O.SUM)
            want = oracle_rs(n, t, dt, O.SUM, p, elems)
            for r in range(n):
                assert same(got[r], want[r]), (dt, n, t, elems, r)


@pytest.mark.parametrize("op", [O.MAX, O.MIN, O.PROD])
@pytest.mark.parametrize("dt", [O.FLOAT32, O.BFLOAT16, O.INT32, O.FLOAT16])
@pytest.mark.parametrize("executor", EXECUTORS)
def test_reduce_scatter_ops(op, dt, executor):
    for n in (3, 8):
        comm = comm_for(n, fused=EXECUTORS[executor])
        elems = 5000
        p = O.random_payload(dt, n * n, elems, 11)
        got = gpu_reduce_scatter(comm, [0] * n, p, elems, dt, op)
        want = oracle_rs(n, O.max_trees(n), dt, op, p, elems)
        for r in range(n):
            assert same(got[r], want[r]), (op, dt, n, r)


@pytest.mark.parametrize("proto", [_lib.PROTO_LL, _lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_PULL])
def test_protocols_forced(proto):
    for n in (2, 5, 8):
        comm = comm_for(n, protocol=proto, fused=-1)
        for elems in (1, 5, 4096, 70001, 300000):
            p = O.random_payload(O.FLOAT32, n, elems, elems)
            got = gpu_allgather(comm, [0] * n, p, elems, O.FLOAT32)
            want = oracle_ag(n, O.max_trees(n), O.FLOAT32, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (proto, n, elems)
            q = O.random_payload(O.BFLOAT16, n * n, elems, elems + 1)
            got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.BFLOAT16, O.SUM)
            want = oracle_rs(n, O.max_trees(n), O.BFLOAT16, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (proto, n, elems)


CONFIG1_EXECUTORS = {"fused": {"fused": 0}, "LL": {"fused": -1, "protocol": _lib.PROTO_LL},
                     "LL32": {"fused": -1, "protocol": _lib.PROTO_LL32},
                     "SIMPLE": {"fused": -1, "protocol": _lib.PROTO_SIMPLE},
                     "PULL": {"fused": -1, "protocol": _lib.PROTO_PULL}}


@pytest.mark.parametrize("executor", CONFIG1_EXECUTORS)
@pytest.mark.parametrize("trees", [1, 2, 4])
def test_config1_exact(trees, executor):
    """BASELINE configs[0] exactly: n = 8, 1 MiB fp32 per rank (262,144 elements), PAT all-gather
    and reduce-scatter(sum) for every valid T (the reference's sweep over T, oracle.cpp:237-282),
    through the fused executor and each transport protocol; bit-exact against the oracle."""
    n, elems = 8, 262144
    comm = comm_for(n, trees=trees, **CONFIG1_EXECUTORS[executor])
    p = O.random_payload(O.FLOAT32, n, elems, 100 + trees)
    got = gpu_allgather(comm, [0] * n, p, elems, O.FLOAT32)
    want = oracle_ag(n, trees, O.FLOAT32, p, elems)
    assert all(same(got[r], want[r]) for r in range(n)), (trees, executor, mismatch(got, want, elems))
    q = O.random_payload(O.FLOAT32, n * n, elems, 200 + trees)
    got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT32, O.SUM)
    want = oracle_rs(n, trees, O.FLOAT32, O.SUM, q, elems)
    assert all(same(got[r], want[r]) for r in range(n)), (trees, executor, mismatch(got, want, elems))
    plan = comm.plan(0, elems, O.FLOAT32)
    assert plan["trees"] == trees and plan["rounds"] == {1: 7, 2: 4, 4: 3}[trees]


@pytest.mark.parametrize("spread", [False, True])
def test_ll32_units_tails_and_alignment(spread):
    """LL32 packs 4-byte units (8-byte units for 8-byte reductions) into 32-byte lines in groups
    of 32; slice tails, element sizes 1..8, 2-, 4- and 8-byte misaligned buffers, in-place
    all-gather and every op stay bit-exact."""
    n = 5
    devices = [r % max(NGPU, 1) for r in range(n)] if spread else [0] * n
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    comm = comm_for(n, devices, protocol=_lib.PROTO_LL32, fused=-1, channels=3, staging_bytes=n * 96 * 1024)
    for dt in (O.INT8, O.FLOAT16, O.BFLOAT16, O.INT32, O.FLOAT32, O.INT64, O.FLOAT64):
        es = _lib.DTYPE_SIZE[dt]
        for elems in (1, 7, 29, 225, 1031, 28673, 100003):
            for pad in (0, 2, 4, 8):
                if pad % es and pad < es:
                    pad = es
                p = O.random_payload(dt, n, elems, elems + pad)
                got = gpu_allgather(comm, devices, p, elems, dt, pad=pad)
                want = oracle_ag(n, O.max_trees(n), dt, p, elems)
                assert all(same(got[r], want[r]) for r in range(n)), ("ag", dt, elems, pad)
                op = [O.SUM, O.MAX, O.PROD, O.MIN][(elems + pad) % 4]
                q = O.random_payload(dt, n * n, elems, elems + pad + 7)
                got = gpu_reduce_scatter(comm, devices, q, elems, dt, op, pad=pad)
                want = oracle_rs(n, O.max_trees(n), dt, op, q, elems)
                assert all(same(got[r], want[r]) for r in range(n)), ("rs", dt, op, elems, pad)
        p = O.random_payload(dt, n, 4099, 77)
        got = gpu_allgather(comm, devices, p, 4099, dt, inplace=True)
        assert all(same(got[r], oracle_ag(n, O.max_trees(n), dt, p, 4099)[r]) for r in range(n)), ("inplace", dt)
    assert comm.plan(0, 1000, O.FLOAT32)["protocol"] == _lib.PROTO_LL32


@pytest.mark.parametrize("executor", EXECUTORS)
def test_misaligned_and_inplace(executor):
    n = 6
    comm = comm_for(n, fused=EXECUTORS[executor])
    for pad in (2, 4, 8):
        for elems in (3, 1001, 100003):
            p = O.random_payload(O.FLOAT16, n, elems, pad)
            got = gpu_allgather(comm, [0] * n, p, elems, O.FLOAT16, pad=pad)
            want = oracle_ag(n, O.max_trees(n), O.FLOAT16, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (pad, elems)
            q = O.random_payload(O.FLOAT16, n * n, elems, pad + 1)
            got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT16, O.SUM, pad=pad)
            want = oracle_rs(n, O.max_trees(n), O.FLOAT16, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (pad, elems)
    for elems in (17, 65536, 300000):
        p = O.random_payload(O.INT32, n, elems, 3)
        got = gpu_allgather(comm, [0] * n, p, elems, O.INT32, inplace=True)
        want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), elems


def test_small_slots_many_pipeline_steps():
    """A tiny staging budget forces many pipeline steps per channel (credit flow control)."""
    n = 8
    comm = comm_for(n, staging_bytes=n * 64 * 1024, channels=4, fused=-1)
    for elems in (1 << 16, 300001):
        p = O.random_payload(O.INT32, n, elems, 5)
        got = gpu_allgather(comm, [0] * n, p, elems, O.INT32)
        want = oracle_ag(n, 4, O.INT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n))
        q = O.random_payload(O.FLOAT32, n * n, elems, 6)
        got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT32, O.SUM)
        want = oracle_rs(n, 4, O.FLOAT32, O.SUM, q, elems)
        assert all(same(got[r], want[r]) for r in range(n))
    plan = comm.plan(1, 300001, O.FLOAT32)
    assert plan["iterations"] > 1 and 1 <= plan["channels"] <= 4
    assert plan["pool_bytes"] <= n * 64 * 1024, plan  # the cap holds for the whole pool, flags included


@pytest.mark.parametrize("executor", EXECUTORS)
def test_back_to_back_calls_mixed_sizes(executor):
    """Iteration counters and credits persist across calls of different sizes and kinds."""
    n = 8
    comm = comm_for(n, fused=EXECUTORS[executor])
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    sizes = [int(x) for x in rng.integers(1, 200000, 40)]
    bufs = []
    for i, elems in enumerate(sizes):
        if i % 2 == 0:
            p = O.random_payload(O.FLOAT32, n, elems, i)
            s = [torch.from_numpy(p[r * elems:(r + 1) * elems].copy()).to(dev) for r in range(n)]
            o = [torch.empty(n * elems, dtype=torch.float32, device=dev) for _ in range(n)]
            comm.all_gather(s, o, elems, O.FLOAT32)
            bufs.append(("ag", elems, p, o, s))
        else:
            p = O.random_payload(O.INT32, n * n, elems, i)
            s = [torch.from_numpy(p[r * n * elems:(r + 1) * n * elems].copy()).to(dev) for r in range(n)]
            o = [torch.empty(elems, dtype=torch.int32, device=dev) for _ in range(n)]
            comm.reduce_scatter(s, o, elems, O.INT32, O.SUM)
            bufs.append(("rs", elems, p, o, s))
    torch.cuda.synchronize()
    comm.raise_async_error()
    for kind, elems, p, o, _ in bufs:
        if kind == "ag":
            want = oracle_ag(n, 4, O.FLOAT32, p, elems)
        else:
            want = oracle_rs(n, 4, O.INT32, O.SUM, p, elems)
        for r in range(n):
            assert same(o[r].cpu().numpy(), want[r]), (kind, elems, r)


@pytest.mark.parametrize("executor", EXECUTORS)
def test_explicit_schedules_generic_executor(executor):
    """Ring / Bruck / single-tree PAT through patAllGatherSchedule / patReduceScatterSchedule."""
    for n in (3, 5, 8):
        comm = comm_for(n, fused=EXECUTORS[executor])
        elems = 3000
        for ag in (S.ring_allgather(n), S.bruck_nearest(n), S.bruck_farthest(n), S.pat_allgather(n, 1)):
            p = O.random_payload(O.FLOAT32, n, elems, 9)
            got = gpu_allgather(comm, [0] * n, p, elems, O.FLOAT32, schedule=ag)
            want, _ = O.run_allgather(ag.encode(), O.FLOAT32, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (n, ag.algorithm)
            rs = S.mirror_schedule(ag)
            q = O.random_payload(O.FLOAT32, n * n, elems, 10)
            got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT32, O.SUM, schedule=rs)
            want, _ = O.run_reduce_scatter(rs.encode(), O.FLOAT32, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (n, rs.algorithm)


@pytest.mark.parametrize("proto", [_lib.PROTO_LL, _lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_PULL])
def test_explicit_schedules_every_protocol(proto):
    """Ring (n-1 rounds, more rounds than pipeline buffers), Bruck and single-tree PAT schedules
    on every transport protocol, across GPUs where there are several, with a small pool so every
    call runs several pipeline steps per channel."""
    for n in (3, 6):
        devices = [r % NGPU for r in range(n)] if NGPU >= 2 else [0] * n
        comm = comm_for(n, devices, protocol=proto, fused=-1, channels=2, staging_bytes=n * 128 * 1024)
        elems = 70001
        for ag in (S.ring_allgather(n), S.bruck_nearest(n), S.pat_allgather(n, 1)):
            p = O.random_payload(O.INT32, n, elems, 31)
            got = gpu_allgather(comm, devices, p, elems, O.INT32, schedule=ag)
            want, _ = O.run_allgather(ag.encode(), O.INT32, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (proto, n, ag.algorithm)
            rs = S.mirror_schedule(ag)
            q = O.random_payload(O.BFLOAT16, n * n, elems, 32)
            got = gpu_reduce_scatter(comm, devices, q, elems, O.BFLOAT16, O.SUM, schedule=rs)
            want, _ = O.run_reduce_scatter(rs.encode(), O.BFLOAT16, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (proto, n, rs.algorithm)


@pytest.mark.parametrize("executor", EXECUTORS)
def test_large_property_checks(executor):
    """Full-size properties: AG output = concatenation; RS int32 = column
    sums mod 2^32; RS fp32 sampled columns = closed-form PAT tree."""
    n = 8
    comm = comm_for(n, fused=EXECUTORS[executor])
    dev = torch.device("cuda:0")
    elems = 8 << 20  # 32 MiB fp32 per rank
    g = torch.Generator(device=dev).manual_seed(0)
    sends = [torch.randint(-2**31, 2**31 - 1, (elems,), dtype=torch.int32, device=dev, generator=g) for _ in range(n)]
    outs = [torch.empty(n * elems, dtype=torch.int32, device=dev) for _ in range(n)]
    comm.all_gather(sends, outs, elems, O.INT32)
    torch.cuda.synchronize()
    cat = torch.cat(sends)
    for r in range(n):
        assert torch.equal(outs[r], cat)
    del outs, cat
    rs_elems = 2 << 20
    rs_send = [torch.randint(-2**31, 2**31 - 1, (n * rs_elems,), dtype=torch.int32, device=dev, generator=g)
               for _ in range(n)]
    rs_out = [torch.empty(rs_elems, dtype=torch.int32, device=dev) for _ in range(n)]
    comm.reduce_scatter(rs_send, rs_out, rs_elems, O.INT32, O.SUM)
    torch.cuda.synchronize()
    stack = torch.stack(rs_send).view(n, n, rs_elems).to(torch.int64)
    for r in range(n):
        want = stack[:, r, :].sum(0)
        want = ((want + 2**31) % 2**32 - 2**31).to(torch.int32)
        assert torch.equal(rs_out[r], want)
    f_send = [torch.rand(n * rs_elems, device=dev, generator=g) for _ in range(n)]
    f_out = [torch.empty(rs_elems, device=dev) for _ in range(n)]
    comm.reduce_scatter(f_send, f_out, rs_elems, O.FLOAT32, O.SUM)
    torch.cuda.synchronize()
    fs = torch.stack(f_send).view(n, n, rs_elems)
    for r in range(n):
        # every element: the closed-form PAT tree evaluated with torch fp32 adds,
        # each an IEEE round-to-nearest add like the kernel's, so the comparison is bit-exact
        want = tree_torch(n, [fs[(r + j) % n, r] for j in range(n)])
        assert torch.equal(f_out[r].view(torch.int32), want.view(torch.int32)), r
    # spot-check the torch tree itself against the C oracle's closed form
    cols = np.random.default_rng(1).integers(0, rs_elems, 16)
    fsn = fs.cpu().numpy()
    for e in cols:
        col = np.array([fsn[(0 + j) % n, 0, e] for j in range(n)], np.float32)
        assert O.tree_fold(n, O.FLOAT32, O.SUM, col) == f_out[0][e].item()


def tree_torch(n, x):
    """The PAT reduce-scatter fold tree for n ranks, accumulator on the left."""
    trees = {
        1: lambda x: x[0],
        2: lambda x: x[0] + x[1],
        3: lambda x: (x[0] + x[1]) + x[2],
        4: lambda x: (x[0] + x[1]) + (x[3] + x[2]),
        5: lambda x: ((x[0] + x[1]) + (x[3] + x[2])) + x[4],
        6: lambda x: ((x[0] + x[1]) + (x[3] + x[2])) + (x[5] + x[4]),
        7: lambda x: ((x[0] + x[1]) + (x[3] + x[2])) + ((x[5] + x[6]) + x[4]),
        8: lambda x: ((x[0] + x[1]) + (x[3] + x[2])) + ((x[5] + (x[7] + x[6])) + x[4]),
    }
    return trees[n](x)


# ------------------------------------------------------------------ multiple GPUs (NVLink peers)

@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8])
def test_multi_gpu_parity(n):
    devices = [r % NGPU for r in range(n)]
    if n <= NGPU:
        devices = list(range(n))
    comm = comm_for(n, devices)
    for elems in (1, 999, 65536, 1 << 20):
        p = O.random_payload(O.FLOAT32, n, elems, elems)
        got = gpu_allgather(comm, devices, p, elems, O.FLOAT32)
        want = oracle_ag(n, O.max_trees(n), O.FLOAT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (n, elems)
        for dt in (O.INT32, O.BFLOAT16):
            q = O.random_payload(dt, n * n, elems, elems + 3)
            got = gpu_reduce_scatter(comm, devices, q, elems, dt, O.SUM)
            want = oracle_rs(n, O.max_trees(n), dt, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (n, elems, dt)


def test_no_async_error_left():
    for c in _COMMS.values():
        assert c.async_error() == 0


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("proto", [_lib.PROTO_LL, _lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_PULL])
@pytest.mark.parametrize("n", [2, 3, 4, 6, 8])
def test_multi_gpu_bulk_protocols(n, proto):
    """SIMPLE (pushed slices through the inboxes) and PULL (receivers read the peers' buffers)
    across NVLink, with a small pool so reduce-scatter staging credits cycle many times."""
    devices = list(range(n)) if n <= NGPU else [r % NGPU for r in range(n)]
    comm = comm_for(n, devices, protocol=proto, staging_bytes=n * 256 * 1024, channels=8)
    for elems in (3, 70001, 600000):
        p = O.random_payload(O.FLOAT32, n, elems, elems + n)
        got = gpu_allgather(comm, devices, p, elems, O.FLOAT32)
        want = oracle_ag(n, O.max_trees(n), O.FLOAT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (n, elems)
        for dt, op in ((O.BFLOAT16, O.SUM), (O.FLOAT32, O.SUM), (O.INT32, O.MAX)):
            q = O.random_payload(dt, n * n, elems, elems + 5)
            got = gpu_reduce_scatter(comm, devices, q, elems, dt, op)
            want = oracle_rs(n, O.max_trees(n), dt, op, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (n, elems, dt, op)


@pytest.mark.parametrize("trees", [1, 2])
def test_pull_single_tree_schedules(trees):
    """PULL with T < max_trees: more rounds than pipeline buffers (no skew), same results."""
    n = 8
    comm = comm_for(n, protocol=_lib.PROTO_PULL, fused=-1, trees=trees, staging_bytes=n * 128 * 1024, channels=4)
    for elems in (5, 100003):
        p = O.random_payload(O.INT32, n, elems, 21)
        got = gpu_allgather(comm, [0] * n, p, elems, O.INT32)
        want = oracle_ag(n, trees, O.INT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (trees, elems)
        q = O.random_payload(O.FLOAT32, n * n, elems, 22)
        got = gpu_reduce_scatter(comm, [0] * n, q, elems, O.FLOAT32, O.SUM)
        want = oracle_rs(n, trees, O.FLOAT32, O.SUM, q, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (trees, elems)


@pytest.mark.parametrize("depth", [0, 2])
@pytest.mark.parametrize("spread", [False, True])
def test_protocol_switches_share_no_inbox_state(spread, depth):
    """One communicator whose calls alternate LL / bulk by size: the polling protocol has its
    own inbox region, so payload words a bulk protocol left behind can never pass for a flag. The int32 payload holds small step-counter-like values to make a collision
    likely if the regions were shared."""
    n = 4
    devices = [r % max(NGPU, 1) for r in range(n)] if spread else [0] * n
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    comm = comm_for(n, devices, fused=-1, channels=2, staging_bytes=n * 32 * 1024, ll_threshold=16384, depth=depth)
    for it in range(24):
        elems = [200, 5000, 300000, 3000][it % 4]  # LL, bulk, bulk (RS: PULL), LL (4-byte elements)
        p = (np.arange(n * elems, dtype=np.int64) % 64 + 1 + it).astype(np.int32)
        got = gpu_allgather(comm, devices, p, elems, O.INT32)
        want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (it, elems, mismatch(got, want, elems))
        q = (np.arange(n * n * elems, dtype=np.int64) % 64 + it).astype(np.int32)
        got = gpu_reduce_scatter(comm, devices, q, elems, O.INT32, O.SUM)
        want = oracle_rs(n, O.max_trees(n), O.INT32, O.SUM, q, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (it, elems, mismatch(got, want, elems))
    plans = [comm.plan(k, e, O.INT32)["protocol"] for k in (0, 1) for e in (200, 5000, 300000)]
    assert plans == [_lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_SIMPLE,
                     _lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_PULL], plans


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_cost_model_protocol_choice():
    """Without an explicit ll_threshold the calibrated alpha-beta model picks LL32 or the bulk
    protocol (comm.cpp: predict_us); the crossovers it implies match the forced sweeps
    (profiles/r01*_forced_n*_p*.jsonl, r02_forced_n*_p*.jsonl: no LL from 256 KiB)."""
    cases = [(2, 64 << 10, _lib.PROTO_LL), (2, 128 << 10, _lib.PROTO_LL), (2, 256 << 10, _lib.PROTO_LL32),
             (2, 2 << 20, _lib.PROTO_LL32), (2, 16 << 20, _lib.PROTO_LL32), (2, 64 << 20, _lib.PROTO_SIMPLE)]
    if NGPU >= 4:
        cases += [(4, 1 << 20, _lib.PROTO_LL32), (4, 16 << 20, _lib.PROTO_LL32), (4, 32 << 20, _lib.PROTO_SIMPLE)]
    for n, nbytes, want in cases:
        comm = comm_for(n, list(range(n)))
        plan = comm.plan(0, nbytes // 4, O.FLOAT32)
        assert plan["protocol"] == want, (n, nbytes, plan)
        assert plan["predicted_us"] > 0


def test_schedule_imported_from_json_runs_on_gpu():
    """§8 f2: a schedule read from the reference's JSON format runs on the generic executor; an
    invalid one is refused with the reference's InvalidScheduleError before any launch."""
    n = 8
    comm = comm_for(n, fused=-1)
    for ag in (S.pat_allgather(n, 1), S.bruck_nearest(n)):
        imported = S.schedule_from_json(S.schedule_to_json(ag))
        p = O.random_payload(O.INT32, n, 999, 5)
        got = gpu_allgather(comm, [0] * n, p, 999, O.INT32, schedule=imported)
        want, _ = O.run_allgather(ag.encode(), O.INT32, p, 999)
        assert all(same(got[r], want[r]) for r in range(n))
    partial = S.schedule_from_json('{"algorithm": "pat", "kind": "allgather", "n_ranks": 8, "params": '
                                   '{"trees": 2, "buffer_slots": 4}, "rounds": [{"round": 0, "dim": 2, '
                                   '"split": 0, "peer": 4, "chunks": [0]}]}')
    with pytest.raises(PatError) as e:
        gpu_allgather(comm, [0] * n, O.random_payload(O.INT32, n, 10, 1), 10, O.INT32, schedule=partial)
    assert e.value.kind == "InvalidScheduleError"


def test_randomized_configurations():
    """Fuzz: random rank counts, placements, dtypes, ops, sizes, alignments, protocols and tree
    counts on long-lived communicators, every result bit-exact against the oracle."""
    rng = np.random.default_rng(2506)
    dtypes = [O.INT8, O.UINT8, O.INT32, O.UINT32, O.INT64, O.FLOAT16, O.FLOAT32, O.FLOAT64, O.BFLOAT16]
    for case in range(40):
        n = int(rng.integers(2, 9))
        spread = NGPU >= 2 and rng.random() < 0.5
        devices = [r % NGPU for r in range(n)] if spread else [0] * n
        proto = int(rng.choice([_lib.PROTO_AUTO, _lib.PROTO_LL, _lib.PROTO_LL32, _lib.PROTO_SIMPLE, _lib.PROTO_PULL]))
        trees = int(rng.choice(O.valid_tree_counts(n)))
        comm = comm_for(n, devices, protocol=proto, trees=trees, fused=-1 if rng.random() < 0.7 else 0,
                        channels=int(rng.choice([1, 3, 8, 32])), staging_bytes=n * int(rng.choice([64, 512])) * 1024)
        dt = int(rng.choice(dtypes))
        es = _lib.DTYPE_SIZE[dt]
        elems = int(rng.choice([1, 3, 17, 1000, 4099, 65536, 200003]))
        pad = int(rng.choice([0, es, 16]))
        p = O.random_payload(dt, n, elems, case)
        got = gpu_allgather(comm, devices, p, elems, dt, pad=pad)
        want = oracle_ag(n, trees, dt, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), ("ag", case, n, devices, proto, trees, dt, elems, pad)
        op = int(rng.choice([O.SUM, O.PROD, O.MAX, O.MIN]))
        q = O.random_payload(dt, n * n, elems, case + 1000)
        got = gpu_reduce_scatter(comm, devices, q, elems, dt, op, pad=pad)
        want = oracle_rs(n, trees, dt, op, q, elems)
        assert all(same(got[r], want[r]) for r in range(n)), ("rs", case, n, devices, proto, trees, dt, op, elems, pad)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_one_process_graph_capture_and_eager_launch_threads():
    """One process over several GPUs: eager calls submit through the per-device launch threads,
    calls captured into per-device CUDA graphs (relaxed, concurrent captures) submit inline;
    both replay bit-exact."""
    n = min(NGPU, 4)
    devices = list(range(n))
    comm = comm_for(n, devices)
    elems = 70001
    p = O.random_payload(O.INT32, n, elems, 41)
    want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
    sends = [torch.from_numpy(p[r * elems:(r + 1) * elems].copy()).to(f"cuda:{r}") for r in range(n)]
    recvs = [torch.zeros(n * elems, dtype=torch.int32, device=f"cuda:{r}") for r in range(n)]
    streams = [torch.cuda.Stream(r) for r in range(n)]
    for _ in range(3):  # eager, launch threads
        comm.all_gather(sends, recvs, elems, O.INT32, streams=streams)
    for r in range(n):
        torch.cuda.synchronize(r)
        assert same(recvs[r].cpu().numpy(), want[r])
        recvs[r].zero_()
    graphs = [torch.cuda.CUDAGraph() for _ in range(n)]
    for r in range(n):
        with torch.cuda.device(r):
            torch.cuda.set_stream(streams[r])
            graphs[r].capture_begin(capture_error_mode="relaxed")
    for _ in range(4):
        comm.all_gather(sends, recvs, elems, O.INT32, streams=streams)
    for r in range(n):
        with torch.cuda.device(r):
            graphs[r].capture_end()
            torch.cuda.set_stream(torch.cuda.default_stream(r))
    for r in range(n):
        torch.cuda.synchronize(r)
        recvs[r].zero_()
        torch.cuda.synchronize(r)
    for _ in range(2):
        for r in range(n):
            with torch.cuda.device(r), torch.cuda.stream(streams[r]):
                graphs[r].replay()
    for r in range(n):
        torch.cuda.synchronize(r)
        assert same(recvs[r].cpu().numpy(), want[r]), r
    comm.raise_async_error()


@pytest.mark.parametrize("spread", [False, True])
def test_bulk_after_polling_call_single_tree(spread):
    """A staged SIMPLE call right after a polling (LL32) call, with the skew at its deepest
    (single-tree PAT, n-1 rounds, depth = rounds): the bulk sender's credit for step base+depth-1
    needs the polling call's last done(step), which that call defers to the next kernel's entry —
    every protocol must publish it there, or sender and receiver wait on each other (regression:
    timed out before transport.cuh published it for bulk kernels)."""
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    n = 4
    devices = [r % max(NGPU, 1) for r in range(n)] if spread else [0] * n
    comm = comm_for(n, devices, fused=-1, direct=-1, depth=3, ll_threshold=1 << 16, channels=4)
    sched_ag = S.pat_allgather(n, 1)
    sched_rs = S.pat_reduce_scatter(n, 1)
    for it in range(12):
        elems = [1000, 200000][it % 2]  # LL32, then staged SIMPLE
        p = (np.arange(n * elems, dtype=np.int64) % 97 + it).astype(np.int32)
        got = gpu_allgather(comm, devices, p, elems, O.INT32, schedule=sched_ag)
        want = oracle_ag(n, 1, O.INT32, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (it, mismatch(got, want, elems))
        q = (np.arange(n * n * elems, dtype=np.int64) % 89 + it).astype(np.int32)
        got = gpu_reduce_scatter(comm, devices, q, elems, O.INT32, O.SUM, schedule=sched_rs)
        want = oracle_rs(n, 1, O.INT32, O.SUM, q, elems)
        assert all(same(got[r], want[r]) for r in range(n)), (it, mismatch(got, want, elems))

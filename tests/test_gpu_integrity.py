"""GPU tests of the transport's integrity rules:

* LL32 accepts a line only when its check word matches its payload (a torn or stale line is
  polled again, never consumed) — tests/cpp/ll32_tear.cu drives ld_line32 directly;
* the 32-bit line flags survive the wrap of the step counter: receivers re-stamp their polling
  buffers once per epoch (transport.cuh, epoch_clean); exercised with 16-step epochs and with
  step counters started just below 2^32;
* one-device communicators allocate no inbox pool until a transport launch needs one;
* a 12 MiB staging cap (3 slots x 4 MiB) holds and stays bit-exact.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import PatComm, _lib  # noqa: E402
from paper_2506_20252_b200 import schedule as S  # noqa: E402

from test_gpu_parity import gpu_allgather, gpu_reduce_scatter, oracle_ag, oracle_rs, same  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def test_ll32_rejects_torn_and_stale_lines(tmp_path):
    exe = tmp_path / "ll32_tear"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++20",
                    "--expt-relaxed-constexpr", "-o", str(exe), os.path.join(ROOT, "tests", "cpp", "ll32_tear.cu")],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("0 failures")


class env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _mixed_calls(comm, devices, calls, seed):
    """Back-to-back all-gathers / reduce-scatters whose sizes switch between LL, LL32 and the
    bulk protocols; every result bit-exact."""
    n = len(devices)
    rng = np.random.default_rng(seed)
    for i in range(calls):
        elems = int(rng.choice([3, 700, 9000, 70001, 300000]))
        dt = [O.INT32, O.FLOAT32, O.BFLOAT16][i % 3]
        p = O.random_payload(dt, n, elems, seed + i)
        got = gpu_allgather(comm, devices, p, elems, dt)
        want = oracle_ag(n, O.max_trees(n), dt, p, elems)
        assert all(same(got[r], want[r]) for r in range(n)), ("ag", i, elems, dt)
        q = O.random_payload(dt, n * n, elems, seed + 1000 + i)
        got = gpu_reduce_scatter(comm, devices, q, elems, dt, O.SUM)
        want = oracle_rs(n, O.max_trees(n), dt, O.SUM, q, elems)
        assert all(same(got[r], want[r]) for r in range(n)), ("rs", i, elems, dt)


@pytest.mark.parametrize("spread", [False, True])
def test_epoch_restamp_every_16_steps(spread):
    if spread and NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    n = 4
    devices = [r % NGPU for r in range(n)] if spread else [0] * n
    with env(PAT_EPOCH_SHIFT=4):
        comm = PatComm.init_all(n, devices, fused=-1, channels=4, staging_bytes=n * 256 * 1024)
    try:
        _mixed_calls(comm, devices, 40, 7)
        comm.raise_async_error()
    finally:
        comm.destroy()


@pytest.mark.parametrize("proto", [_lib.PROTO_LL, _lib.PROTO_LL32, _lib.PROTO_AUTO])
def test_step_counter_crosses_2_pow_32(proto):
    """Counters start 120 steps below 2^32: the calls cross uint32(g + 1) = 0, where a zeroed or
    2^32-steps-old line would pass for the current step without the epoch re-stamp."""
    n = 4
    devices = list(range(n)) if NGPU >= n else [0] * n
    with env(PAT_ITER_START=(1 << 32) - 120):
        comm = PatComm.init_all(n, devices, fused=-1, protocol=proto, channels=2, staging_bytes=n * 256 * 1024)
    try:
        rng = np.random.default_rng(proto)
        for i in range(100):  # 1-4 steps per call and channel
            elems = int(rng.choice([5, 2000, 20000]))
            p = O.random_payload(O.INT32, n, elems, i)
            got = gpu_allgather(comm, devices, p, elems, O.INT32)
            want = oracle_ag(n, O.max_trees(n), O.INT32, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (i, elems)
            q = O.random_payload(O.FLOAT32, n * n, elems, 500 + i)
            got = gpu_reduce_scatter(comm, devices, q, elems, O.FLOAT32, O.SUM)
            want = oracle_rs(n, O.max_trees(n), O.FLOAT32, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (i, elems)
        comm.raise_async_error()
    finally:
        comm.destroy()


def test_one_device_pools_are_lazy():
    n = 8
    comm = PatComm.init_all(n, [0] * n)
    try:
        for elems in (1000, 300000):
            p = O.random_payload(O.FLOAT32, n, elems, 3)
            assert all(same(a, b) for a, b in zip(gpu_allgather(comm, [0] * n, p, elems, O.FLOAT32),
                                                  oracle_ag(n, 4, O.FLOAT32, p, elems)))
        info = comm.pool_info()
        assert info["allocated_bytes"] == 0 and not info["pools_allocated"], info
        assert comm.plan(0, 1000, O.FLOAT32)["protocol"] == _lib.PROTO_FUSED
        # a ring schedule is not the fused executor's tree: the transport runs, pools appear
        ring = S.mirror_schedule(S.ring_allgather(n))
        q = O.random_payload(O.FLOAT32, n * n, 5000, 4)
        got = gpu_reduce_scatter(comm, [0] * n, q, 5000, O.FLOAT32, O.SUM, schedule=ring)
        want, _ = O.run_reduce_scatter(ring.encode(), O.FLOAT32, O.SUM, q, 5000)
        assert all(same(got[r], want[r]) for r in range(n))
        info = comm.pool_info()
        assert info["pools_allocated"] and info["allocated_bytes"] == n * info["pool_bytes_per_rank"], info
    finally:
        comm.destroy()


def test_staging_cap_12mib_holds_and_stays_exact():
    """SURVEY §8d config 5's example cap (3 slots x 4 MiB) on the ZeRO-3 shape's protocols."""
    n = 4
    devices = list(range(n)) if NGPU >= n else [0] * n
    cap = 12 << 20
    comm = PatComm.init_all(n, devices, fused=-1, staging_bytes=cap)
    try:
        info = comm.pool_info()
        assert info["pool_bytes_per_rank"] <= cap, info
        for dt, elems in ((O.BFLOAT16, 3 << 20), (O.INT32, 1 << 20), (O.FLOAT32, 77777)):
            p = O.random_payload(dt, n, elems, elems)
            got = gpu_allgather(comm, devices, p, elems, dt)
            want = oracle_ag(n, O.max_trees(n), dt, p, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (dt, elems)
            q = O.random_payload(dt, n * n, elems, elems + 1)
            got = gpu_reduce_scatter(comm, devices, q, elems, dt, O.SUM)
            want = oracle_rs(n, O.max_trees(n), dt, O.SUM, q, elems)
            assert all(same(got[r], want[r]) for r in range(n)), (dt, elems)
            for k in (0, 1):
                plan = comm.plan(k, elems, dt)
                assert plan["staging_bytes_used"] <= cap, plan
        comm.raise_async_error()
    finally:
        comm.destroy()

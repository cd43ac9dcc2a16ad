"""The Python collectives check tensor arguments before launching (a too-small, non-contiguous or
misplaced buffer would make the kernels write outside it): PayloadShapeError / InvalidArgument,
raised on the host; raw pointers pass unchecked as at the C ABI; valid calls still bit-exact."""
import pytest


torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_20252_b200 import FLOAT32, SUM, PatComm, PatError  # noqa: E402

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def test_tensor_checks_one_process():
    n, e = 4, 1000
    comm = PatComm.init_all(n, [0] * n)
    try:
        s = [torch.rand(e, device="cuda:0") for _ in range(n)]
        r = [torch.empty(n * e, device="cuda:0") for _ in range(n)]
        short = r[:3] + [torch.empty(n * e - 1, device="cuda:0")]
        with pytest.raises(PatError) as ei:
            comm.all_gather(s, short, e, FLOAT32)
        assert ei.value.kind == "PayloadShapeError"
        strided = r[:3] + [torch.empty(2 * n * e, device="cuda:0")[::2]]
        with pytest.raises(PatError) as ei:
            comm.all_gather(s, strided, e, FLOAT32)
        assert ei.value.kind == "InvalidArgument"
        with pytest.raises(PatError) as ei:
            comm.all_gather(s[:3], r[:3], e, FLOAT32)
        assert ei.value.kind == "InvalidArgument"
        with pytest.raises(PatError) as ei:  # reduce-scatter input: n * count per rank
            comm.reduce_scatter(s, [x[:e] for x in r], e, FLOAT32, SUM)
        assert ei.value.kind == "PayloadShapeError"
        if NGPU > 1:
            with pytest.raises(PatError) as ei:
                comm.all_gather(s[:3] + [s[3].to("cuda:1")], r, e, FLOAT32)
            assert ei.value.kind == "InvalidArgument"
        # the C ABI's own checks (raw pointers): a null buffer, a count whose n * count bytes overflow
        with pytest.raises(PatError) as ei:
            comm.all_gather([x.data_ptr() for x in s[:3]] + [0], [x.data_ptr() for x in r], e, FLOAT32)
        assert ei.value.kind == "InvalidArgument"
        with pytest.raises(PatError) as ei:
            comm.all_gather([x.data_ptr() for x in s], [x.data_ptr() for x in r], 1 << 61, FLOAT32)
        assert ei.value.kind == "InvalidArgument"
        comm.all_gather(s, r, e, FLOAT32)  # nothing was launched by the refused calls
        torch.cuda.synchronize()
        want = torch.cat([x.cpu() for x in s])
        for x in r:
            assert torch.equal(x.cpu(), want)
        comm.validate_tensors = False  # opt-out: sizes are the caller's responsibility
        comm.all_gather(s, r, e, FLOAT32)
        torch.cuda.synchronize()
        comm.raise_async_error()
    finally:
        comm.destroy()


@pytest.mark.parametrize("fused", [0, -1])
def test_single_rank(fused):
    """n = 1 (the reference accepts it: zero rounds): all-gather and reduce-scatter are copies."""
    comm = PatComm.init_all(1, [0], fused=fused)
    try:
        for e in (1, 3000, 1 << 20):
            s = torch.rand(e, device="cuda:0")
            r = torch.empty(e, device="cuda:0")
            comm.all_gather([s], [r], e, FLOAT32)
            torch.cuda.synchronize()
            assert torch.equal(r, s)
            r.zero_()
            comm.reduce_scatter([s], [r], e, FLOAT32, SUM)
            torch.cuda.synchronize()
            assert torch.equal(r, s)
        comm.raise_async_error()
    finally:
        comm.destroy()

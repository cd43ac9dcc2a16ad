"""Host-side argument checks of the Python collectives (no GPU: a communicator shell with the
device layout of 2 local ranks; CPU tensors report device -1)."""
import pytest

torch = pytest.importorskip("torch")

from paper_2506_20252_b200 import PatComm, PatError  # noqa: E402


def shell(devices):
    c = object.__new__(PatComm)
    c.local_ranks = list(range(len(devices)))
    c.devices = list(devices)
    c.nranks = 4
    return c


def test_tensor_checks():
    c = shell([-1, -1])  # CPU tensors: get_device() == -1
    ok = [torch.empty(16), torch.empty(16)]
    c._check_tensors(ok, 64, "x")
    with pytest.raises(PatError) as ei:
        c._check_tensors([ok[0], torch.empty(15)], 64, "x")
    assert ei.value.kind == "PayloadShapeError"
    with pytest.raises(PatError) as ei:
        c._check_tensors([ok[0], torch.empty(32)[::2]], 64, "x")
    assert ei.value.kind == "InvalidArgument"
    with pytest.raises(PatError) as ei:
        c._check_tensors(ok[:1], 64, "x")
    assert ei.value.kind == "InvalidArgument"
    c._check_tensors([ok[0], 12345], 64, "x")  # raw pointers pass unchecked
    with pytest.raises(PatError) as ei:
        shell([-1, 0])._check_tensors(ok, 64, "x")
    assert ei.value.kind == "InvalidArgument"
    c.validate_tensors = False
    c._check_tensors([ok[0], torch.empty(1)], 64, "x")
    with pytest.raises(PatError):  # the count of buffers is always checked
        c._check_tensors(ok[:1], 64, "x")

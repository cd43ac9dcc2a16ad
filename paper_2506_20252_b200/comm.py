"""Communicators and collectives over the C ABI (include/pat_b200.h).

Two ways to build a communicator, matching the north-star process models:

* ``PatComm.init_all(n, devices)`` — one process drives all ranks (the reference's in-process
  ranks, ``ncclCommInitAll``). ``devices`` may repeat a GPU: its ranks then run inside one
  cooperative kernel ("local mode", used for n > #GPUs and for the 1-GPU HBM roofline).
* ``PatComm.init_rank(n, rank, device, exchange)`` / ``from_process_group()`` — one process
  per rank (torchrun). Each rank exports a 128-byte handle; ``exchange`` all-gathers them
  (torch.distributed, any backend) and the peers' inbox pools are mapped with CUDA IPC.

Buffers are passed as raw device pointers (ints) or torch tensors; torch is plumbing only.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional, Sequence

from . import _lib
from ._lib import Config, PatError, PlanInfo, check, lib, ptr_array

try:  # torch is optional for the pointer-level API
    import torch

    TORCH_DTYPES = {
        torch.int8: _lib.INT8, torch.uint8: _lib.UINT8, torch.int32: _lib.INT32, torch.int64: _lib.INT64,
        torch.float16: _lib.FLOAT16, torch.float32: _lib.FLOAT32, torch.float64: _lib.FLOAT64,
        torch.bfloat16: _lib.BFLOAT16,
    }
    for _name, _code in (("uint32", _lib.UINT32), ("uint64", _lib.UINT64)):
        if hasattr(torch, _name):
            TORCH_DTYPES[getattr(torch, _name)] = _code
except ImportError:  # pragma: no cover
    torch = None
    TORCH_DTYPES = {}


def make_config(**kw) -> Config:
    c = Config()
    lib().patConfigInit(ctypes.byref(c))
    mapping = {"channels": "max_channels"}
    for k, v in kw.items():
        if v is None:
            continue
        setattr(c, mapping.get(k, k), int(v))
    return c


def _ptr(x) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"expected a device pointer or tensor, got {type(x)}")


def _dtype(dtype, sample) -> int:
    if dtype is None:
        if torch is None or not hasattr(sample, "dtype"):
            raise TypeError("dtype required for raw pointers")
        return TORCH_DTYPES[sample.dtype]
    if torch is not None and isinstance(dtype, torch.dtype):
        return TORCH_DTYPES[dtype]
    return int(dtype)


def make_exchange(group=None) -> Callable[[bytes], list]:
    """All-gather of the per-rank init handles over a torch.distributed group (any backend)."""
    import torch.distributed as dist

    def exchange(mine: bytes) -> list:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, bytes(mine), group=group)
        if any(not isinstance(x, (bytes, bytearray)) or len(x) != _lib.HANDLE_BYTES for x in out):
            raise PatError(4, "handle exchange returned a malformed list")
        return [bytes(x) for x in out]

    return exchange


class group:
    """``with group(): ...`` — patGroupStart / patGroupEnd: the collectives issued inside are launched
    at exit; an all-gather and a reduce-scatter (sum) of one communicator on the same streams run
    as one launch. The calls must be independent; errors surface at exit."""

    def __enter__(self):
        check(lib().patGroupStart(), "patGroupStart")
        return self

    def __exit__(self, exc_type, exc, tb):
        rc = lib().patGroupEnd()
        if exc_type is None:
            check(rc, "patGroupEnd")
        return False


class PatComm:
    # tensors passed to the collectives are checked (size, contiguity, device) before the launch;
    # raw integer pointers are not (as at the C ABI). Set False to skip the checks (~0.5 us/tensor).
    validate_tensors = True

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        n = ctypes.c_int()
        check(lib().patCommCount(self._h, ctypes.byref(n)), "patCommCount")
        self.nranks = n.value
        self._hv = int(handle.value) if handle.value else 0
        nl = ctypes.c_int()
        ranks = (ctypes.c_int * _lib.MAX_RANKS)()
        devs = (ctypes.c_int * _lib.MAX_RANKS)()
        check(lib().patCommLocalRanks(self._h, ctypes.byref(nl), ranks, devs), "patCommLocalRanks")
        self.local_ranks = list(ranks[: nl.value])
        self.devices = list(devs[: nl.value])
        self._fast = _lib.fast()
        self._raw_stream = (getattr(torch._C, "_cuda_getCurrentRawStream", None)
                            if torch is not None and torch.cuda.is_available() else None)

    # ------------------------------------------------------------------ construction
    @classmethod
    def init_all(cls, nranks: int, devices: Optional[Sequence[int]] = None, **config) -> "PatComm":
        h = ctypes.c_void_p()
        cfg = make_config(**config)
        devarr = (ctypes.c_int * nranks)(*devices) if devices is not None else None
        check(lib().patCommInitAll(ctypes.byref(h), nranks, devarr, ctypes.byref(cfg)), "patCommInitAll")
        return cls(h)

    @classmethod
    def init_rank(cls, nranks: int, rank: int, device: int, exchange: Callable[[bytes], list], **config) -> "PatComm":
        """exchange(my_handle_bytes) must return all ranks' handles, rank-ordered."""
        h = ctypes.c_void_p()
        cfg = make_config(**config)
        blob = ctypes.create_string_buffer(_lib.HANDLE_BYTES)
        check(lib().patCommInitRankPrepare(ctypes.byref(h), nranks, rank, device, ctypes.byref(cfg), blob),
              "patCommInitRankPrepare")
        try:
            handles = exchange(bytes(blob.raw))
            if len(handles) != nranks or any(len(x) != _lib.HANDLE_BYTES for x in handles):
                raise PatError(4, "handle exchange returned a malformed list")
            allh = ctypes.create_string_buffer(b"".join(handles), nranks * _lib.HANDLE_BYTES)
            check(lib().patCommInitRankFinish(h, allh), "patCommInitRankFinish")
        except BaseException:
            lib().patCommDestroy(h)
            raise
        c = cls(h)
        c._exchange = exchange
        return c

    @classmethod
    def from_process_group(cls, group=None, device: Optional[int] = None, **config) -> "PatComm":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        return cls.init_rank(world, rank, device, make_exchange(group), **config)

    def destroy(self) -> None:
        if self._h:
            lib().patCommDestroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.destroy()
        except Exception:
            pass

    # ------------------------------------------------------------------ collectives
    def _streams(self, streams):
        if streams is None:
            if torch is not None and torch.cuda.is_available():
                cur = {}  # one current-stream lookup per device, not per local rank
                for d in self.devices:
                    if d not in cur:
                        cur[d] = torch.cuda.current_stream(d).cuda_stream
                streams = [cur[d] for d in self.devices]
            else:
                streams = [0] * len(self.local_ranks)
        return ptr_array([int(getattr(s, "cuda_stream", s)) for s in streams])

    def _fast_streams(self, streams):
        """Stream handles as plain ints for _patfast (one current-stream lookup per device)."""
        if streams is None:
            if self._raw_stream is not None:
                if len(self.devices) == 1:
                    return self._raw_stream(self.devices[0])
                cur = {}
                for d in self.devices:
                    if d not in cur:
                        cur[d] = self._raw_stream(d)
                return [cur[d] for d in self.devices]
            return [0] * len(self.local_ranks)
        return [int(getattr(s, "cuda_stream", s)) for s in streams]

    def _check_tensors(self, bufs, nbytes: int, what: str) -> None:
        """Every tensor in bufs (one per local rank) holds nbytes contiguous bytes on its rank's device."""
        if len(bufs) != len(self.local_ranks):
            raise PatError(4, f"{what}: {len(bufs)} buffers for {len(self.local_ranks)} local ranks")
        if not self.validate_tensors:
            return
        for x, d in zip(bufs, self.devices):
            if type(x) is int:
                continue
            if x.nbytes < nbytes:
                raise PatError(31, f"{what}: a buffer holds {x.nbytes} bytes, the call needs {nbytes}")
            if not x.is_contiguous():
                raise PatError(4, f"{what}: buffers must be contiguous")
            if x.get_device() != d:
                raise PatError(4, f"{what}: a buffer is on device {x.get_device()}, its rank on {d}")

    def all_gather(self, sendbufs, recvbufs, count: Optional[int] = None, dtype=None, streams=None, schedule=None):
        """sendbufs[l] -> recvbufs[l] (n*count, origin order) for every local rank l."""
        dt = _dtype(dtype, sendbufs[0])
        if count is None:
            count = sendbufs[0].numel()
        es = _lib.DTYPE_SIZE.get(dt, 0)  # an unknown dtype is refused by the library
        self._check_tensors(sendbufs, count * es, "all_gather sendbufs")
        self._check_tensors(recvbufs, self.nranks * count * es, "all_gather recvbufs")
        if schedule is None and self._fast is not None and self._h:
            check(self._fast.all_gather(self._hv, [_ptr(x) for x in sendbufs], [_ptr(x) for x in recvbufs], count, dt,
                                        self._fast_streams(streams)), "patAllGather")
            return
        sb, rb = ptr_array([_ptr(x) for x in sendbufs]), ptr_array([_ptr(x) for x in recvbufs])
        if schedule is not None:
            enc = schedule.encode()
            check(lib().patAllGatherSchedule(self._h, enc.ctypes.data_as(_lib.I32P), len(enc), sb, rb, count, dt,
                                             self._streams(streams)), "patAllGatherSchedule")
        else:
            check(lib().patAllGather(self._h, sb, rb, count, dt, self._streams(streams)), "patAllGather")

    def reduce_scatter(self, sendbufs, recvbufs, count: Optional[int] = None, dtype=None, op: int = _lib.SUM,
                       streams=None, schedule=None):
        """sendbufs[l] (n*count, block d -> rank d) reduced into recvbufs[l] (count)."""
        dt = _dtype(dtype, sendbufs[0])
        if count is None:
            count = recvbufs[0].numel()
        es = _lib.DTYPE_SIZE.get(dt, 0)  # an unknown dtype is refused by the library
        self._check_tensors(sendbufs, self.nranks * count * es, "reduce_scatter sendbufs")
        self._check_tensors(recvbufs, count * es, "reduce_scatter recvbufs")
        if schedule is None and self._fast is not None and self._h:
            check(self._fast.reduce_scatter(self._hv, [_ptr(x) for x in sendbufs], [_ptr(x) for x in recvbufs], count,
                                            dt, int(op), self._fast_streams(streams)), "patReduceScatter")
            return
        sb, rb = ptr_array([_ptr(x) for x in sendbufs]), ptr_array([_ptr(x) for x in recvbufs])
        if schedule is not None:
            enc = schedule.encode()
            check(lib().patReduceScatterSchedule(self._h, enc.ctypes.data_as(_lib.I32P), len(enc), sb, rb, count,
                                                 dt, int(op), self._streams(streams)), "patReduceScatterSchedule")
        else:
            check(lib().patReduceScatter(self._h, sb, rb, count, dt, int(op), self._streams(streams)),
                  "patReduceScatter")

    # ---- torch.distributed-shaped forms for one rank per process (ZeRO-3 style callers)
    def all_gather_into_tensor(self, output, input, stream=None):
        """output (n * input.numel(), rank-ordered) <- every rank's input, like
        torch.distributed.all_gather_into_tensor; on `stream` (default: the current stream)."""
        if len(self.local_ranks) != 1:
            raise PatError(5, "all_gather_into_tensor needs a one-rank-per-process communicator")
        if output.numel() != self.nranks * input.numel() or output.dtype != input.dtype:
            raise PatError(31, "all_gather_into_tensor: output must hold nranks * input.numel() of input's dtype")
        self._check_pair(output, input, "all_gather_into_tensor")
        if self._fast is not None and self._h:
            st = self._fast_streams(None if stream is None else [stream])
            check(self._fast.all_gather(self._hv, input.data_ptr(), output.data_ptr(), input.numel(),
                                        TORCH_DTYPES[input.dtype], st if isinstance(st, int) else st[0]),
                  "patAllGather")
            return
        self.all_gather([input], [output], input.numel(), None, None if stream is None else [stream])

    def reduce_scatter_tensor(self, output, input, op: int = _lib.SUM, stream=None):
        """output (input.numel() / n) <- fold of block `rank` of every rank's input, like
        torch.distributed.reduce_scatter_tensor, in the PAT tree order."""
        if len(self.local_ranks) != 1:
            raise PatError(5, "reduce_scatter_tensor needs a one-rank-per-process communicator")
        if input.numel() != self.nranks * output.numel() or output.dtype != input.dtype:
            raise PatError(31, "reduce_scatter_tensor: input must hold nranks * output.numel() of output's dtype")
        self._check_pair(output, input, "reduce_scatter_tensor")
        if self._fast is not None and self._h:
            st = self._fast_streams(None if stream is None else [stream])
            check(self._fast.reduce_scatter(self._hv, input.data_ptr(), output.data_ptr(), output.numel(),
                                            TORCH_DTYPES[output.dtype], int(op), st if isinstance(st, int) else st[0]),
                  "patReduceScatter")
            return
        self.reduce_scatter([input], [output], output.numel(), None, op, None if stream is None else [stream])

    def _check_pair(self, output, input, what: str) -> None:
        if self.validate_tensors and not (output.is_contiguous() and input.is_contiguous() and
                                          output.get_device() == input.get_device() == self.devices[0]):
            raise PatError(4, f"{what}: tensors must be contiguous and on device {self.devices[0]}")

    @staticmethod
    def group() -> "group":
        return group()

    def barrier(self, streams=None) -> None:
        """Device-side barrier over every rank on `streams` (default: the current streams)."""
        check(lib().patCommBarrier(self._h, self._streams(streams)), "patCommBarrier")

    # ---- symmetric windows (one rank per process): zero-copy all-gather / PULL reduce-scatter
    def register(self, buf, nbytes: Optional[int] = None) -> None:
        """Collective: every rank registers a window of the same size (a cudaMalloc'd tensor or
        pointer), in the same order. Calls whose all-gather recvbuf / reduce-scatter sendbuf lie
        inside a window at the same offset on every rank then run zero copy
        (patCommRegisterPrepare/Finish)."""
        exchange = getattr(self, "_exchange", None)
        if exchange is None:
            raise PatError(5, "register needs a one-rank-per-process communicator (init_rank)")
        if nbytes is None:
            nbytes = buf.numel() * buf.element_size()
        blob = ctypes.create_string_buffer(_lib.HANDLE_BYTES)
        check(lib().patCommRegisterPrepare(self._h, _ptr(buf), int(nbytes), blob), "patCommRegisterPrepare")
        handles = exchange(bytes(blob.raw))
        allh = ctypes.create_string_buffer(b"".join(handles), self.nranks * _lib.HANDLE_BYTES)
        check(lib().patCommRegisterFinish(self._h, _ptr(buf), allh), "patCommRegisterFinish")

    def deregister(self, buf) -> None:
        """Local; only after every call that used the window has completed."""
        check(lib().patCommDeregister(self._h, _ptr(buf)), "patCommDeregister")

    def plan(self, kind: int, count: int, dtype) -> dict:
        info = PlanInfo()
        check(lib().patCommPlan(self._h, int(kind), count, _dtype(dtype, None) if dtype is not None else 7,
                                ctypes.byref(info)), "patCommPlan")
        return info.as_dict()

    def pool_info(self) -> dict:
        """Inbox pool layout and what this process has allocated (patCommMemInfo)."""
        info = _lib.MemInfo()
        check(lib().patCommMemInfo(self._h, ctypes.byref(info)), "patCommMemInfo")
        return info.as_dict()

    def trace(self, group: int = 0):
        """Device event trace of the last transport launch (PAT_TRACE=<entries> at init).
        Returns a numpy array [ctas, 2 roles, entries, 2] of (globaltimer ns, code)."""
        import numpy as np

        nb, ctas, ent = ctypes.c_size_t(), ctypes.c_int(), ctypes.c_int()
        lib().patCommTraceRead(self._h, group, None, 0, ctypes.byref(nb), ctypes.byref(ctas), ctypes.byref(ent))
        buf = np.zeros(nb.value // 8, np.uint64)
        check(lib().patCommTraceRead(self._h, group, buf.ctypes.data, nb.value, ctypes.byref(nb),
                                     ctypes.byref(ctas), ctypes.byref(ent)), "patCommTraceRead")
        return buf.reshape(ctas.value, 2, ent.value, 2)

    def device_occupancy(self) -> list:
        """Per local rank: intermediate slots held after every round, as counted by the device in
        the last SIMPLE launch (communicator created with PAT_STATS=1; patCommStatsRead)."""
        buf = (ctypes.c_int32 * (_lib.MAX_RANKS * 8))()
        nl, nr = ctypes.c_int(), ctypes.c_int()
        check(lib().patCommStatsRead(self._h, buf, ctypes.byref(nl), ctypes.byref(nr)), "patCommStatsRead")
        return [list(buf[l * 8:l * 8 + nr.value]) for l in range(nl.value)] if nr.value >= 0 else []

    def async_error(self) -> int:
        e = ctypes.c_int()
        check(lib().patCommGetAsyncError(self._h, ctypes.byref(e)), "patCommGetAsyncError")
        return e.value

    def raise_async_error(self) -> None:
        e = self.async_error()
        if e:
            raise PatError(e, "asynchronous device error")

"""The reference executor's API (run_allgather / run_reduce_scatter over a Payload), on B200.

Reference: /root/reference/proj/include/patsim/simulate.hpp:14-96. Same argument meaning,
same payload layouts and the same typed errors (PayloadShapeError, UnsupportedOpError,
InvalidScheduleError, SimulationError), but the data path is the sm_100a kernels behind
the C ABI: every logical rank's payload is copied to its GPU, the schedule runs through
``patAllGatherSchedule`` / ``patReduceScatterSchedule``, and the outputs are copied back.
By default all ranks are placed on ``cuda:0`` (local mode, one cooperative kernel);
``RunOptions.devices`` spreads them over GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _lib
from .comm import PatComm
from .schedule import CollectiveKind, RelativeSchedule, stats as schedule_stats


class ReduceOp(IntEnum):  # simulate.hpp:14
    WrappingIntSum = 0
    FloatSum = 1


class ExecMode(IntEnum):  # simulate.hpp:16 (the GPU path has one mode; kept for signature parity)
    Lockstep = 0
    Parallel = 1


@dataclass
class RunOptions:  # simulate.hpp:63-67
    mode: ExecMode = ExecMode.Lockstep
    threads: int = 0
    devices: Optional[list] = None   # CUDA device of every rank; None = all on device 0
    config: dict = field(default_factory=dict)


@dataclass
class Payload:  # simulate.hpp:36-41
    n_ranks: int = 0
    elements_per_chunk: int = 0
    chunks: list = field(default_factory=list)


@dataclass
class CollectiveResult:  # simulate.hpp:55-60
    outputs: list
    stats: dict


class SimulationError(_lib.PatError):
    pass


def _raise(code: int, msg: str):
    raise _lib.PatError(code, msg)


_COMMS: dict = {}


def _comm(n: int, devices, config: dict) -> PatComm:
    key = (n, tuple(devices), tuple(sorted(config.items())))
    if key not in _COMMS:
        _COMMS[key] = PatComm.init_all(n, devices, **config)
    return _COMMS[key]


def _ensure_payload(sched: RelativeSchedule, payload: Payload, reduce_scatter: bool) -> np.dtype:
    # ensure_payload (simulate.cpp:87-107)
    want = sched.n_ranks * sched.n_ranks if reduce_scatter else sched.n_ranks
    if payload.n_ranks != sched.n_ranks:
        _raise(31, f"payload is for {payload.n_ranks} ranks, schedule for {sched.n_ranks}")
    if payload.elements_per_chunk < 1:
        _raise(31, "elements_per_chunk must be >= 1")
    if len(payload.chunks) != want:
        _raise(31, f"payload has {len(payload.chunks)} chunks, expected {want}")
    dts = {np.asarray(c).dtype for c in payload.chunks}
    for c in payload.chunks:
        if np.asarray(c).size != payload.elements_per_chunk:
            _raise(31, "all chunks must have elements_per_chunk elements")
    if len(dts) != 1:
        _raise(31, "all chunks must share one dtype")
    return dts.pop()


_NP_TO_PAT = {np.dtype(np.int64): _lib.INT64, np.dtype(np.float64): _lib.FLOAT64,
              np.dtype(np.int32): _lib.INT32, np.dtype(np.float32): _lib.FLOAT32,
              np.dtype(np.uint32): _lib.UINT32, np.dtype(np.uint64): _lib.UINT64,
              np.dtype(np.int8): _lib.INT8, np.dtype(np.uint8): _lib.UINT8}


def _run(kind: int, sched: RelativeSchedule, payload: Payload, dtype: int, op: int, options: RunOptions):
    import torch

    n = sched.n_ranks
    elems = payload.elements_per_chunk
    devices = options.devices or [0] * n
    comm = _comm(n, devices, dict(options.config))
    per_rank = n if kind == CollectiveKind.ReduceScatter else 1
    host = np.stack([np.asarray(c) for c in payload.chunks]).reshape(n, per_rank * elems)
    sends = [torch.from_numpy(np.ascontiguousarray(host[r]).view(np.uint8).copy()).to(f"cuda:{devices[r]}")
             for r in range(n)]
    out_elems = n * elems if kind == CollectiveKind.AllGather else elems
    recvs = [torch.zeros(out_elems * host.dtype.itemsize, dtype=torch.int8, device=f"cuda:{devices[r]}")
             for r in range(n)]
    if kind == CollectiveKind.AllGather:
        comm.all_gather(sends, recvs, elems, dtype, schedule=sched)
    else:
        comm.reduce_scatter(sends, recvs, elems, dtype, op, schedule=sched)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    comm.raise_async_error()
    outputs = [r.cpu().numpy().view(host.dtype).copy() for r in recvs]
    st = schedule_stats(sched, elems * 8)  # the reference counts 8-byte elements (simulate.cpp:17)
    return CollectiveResult(outputs, st)


def run_allgather(sched: RelativeSchedule, payload: Payload, options: Optional[RunOptions] = None):
    """simulate.hpp:78-84: outputs[r] = the n chunks in origin order."""
    options = options or RunOptions()
    if sched.kind != CollectiveKind.AllGather:
        _raise(30, "schedule kind is reducescatter, expected allgather")
    dt = _ensure_payload(sched, payload, False)
    code = _NP_TO_PAT.get(dt)
    if code is None:
        _raise(32, f"unsupported payload dtype {dt}")
    return _run(CollectiveKind.AllGather, sched, payload, code, _lib.SUM, options)


def run_reduce_scatter(sched: RelativeSchedule, payload: Payload, op: ReduceOp, options: Optional[RunOptions] = None):
    """simulate.hpp:93-96: outputs[r] = reduction of chunks[s*n + r] in the PAT tree order."""
    options = options or RunOptions()
    dt = _ensure_payload(sched, payload, True) if payload.chunks else None
    # op/type pairing (simulate.cpp:316-332)
    if dt == np.dtype(np.int64) and op != ReduceOp.WrappingIntSum:
        _raise(32, "UnsupportedOp: integer payloads reduce with WrappingIntSum")
    if dt == np.dtype(np.float64) and op != ReduceOp.FloatSum:
        _raise(32, "UnsupportedOp: float payloads reduce with FloatSum")
    if sched.kind != CollectiveKind.ReduceScatter:
        _raise(30, "schedule kind is allgather, expected reducescatter")
    code = _NP_TO_PAT.get(dt)
    if code is None:
        _raise(32, f"unsupported payload dtype {dt}")
    return _run(CollectiveKind.ReduceScatter, sched, payload, code, _lib.SUM, options)

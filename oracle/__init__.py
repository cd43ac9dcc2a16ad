"""ctypes view of the parity checker — TEST INFRASTRUCTURE ONLY.

Two libraries live here:

* ``oracle/build/libpat_oracle.so`` — the C restatement of the reference's PAT path
  (``oracle/pat_oracle.c``; every function cites the reference file:line it follows).
* ``oracle/_ref/libpatsim_ref.so`` — the reference itself, compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` (present only where it was built;
  it travels to the GPU box as a prebuilt file).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) import this package, and only as the checker / CPU baseline.
The product (``paper_2506_20252_b200``) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libpat_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpatsim_ref.so")

ALLGATHER, REDUCESCATTER = 0, 1
RING, BRUCK_NEAREST, BRUCK_FARTHEST, RECURSIVE_DOUBLING, PAT = range(5)
INT8, UINT8, INT32, UINT32, INT64, UINT64, FLOAT16, FLOAT32, FLOAT64, BFLOAT16 = range(10)
SUM, PROD, MAX, MIN = range(4)

# numpy storage dtype per wire dtype (fp16/bf16 are carried as uint16 bit patterns)
NP_DTYPE = {
    INT8: np.int8, UINT8: np.uint8, INT32: np.int32, UINT32: np.uint32, INT64: np.int64,
    UINT64: np.uint64, FLOAT16: np.uint16, FLOAT32: np.float32, FLOAT64: np.float64,
    BFLOAT16: np.uint16,
}

ERRORS = {
    1: "ScheduleError", 2: "NonPowerOfTwoError", 3: "InvalidTreeCountError",
    4: "BufferTooSmallError", 5: "RankOutOfRangeError", 10: "SimulationError",
    11: "PayloadShapeError", 12: "UnsupportedOpError", 13: "InvalidScheduleError",
    20: "CapacityError", 30: "ParseError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.kind = ERRORS.get(code, f"error{code}")
        super().__init__(f"{where}: {self.kind}")


class PoStats(ctypes.Structure):
    _fields_ = [
        ("rounds", ctypes.c_int32),
        ("max_chunks_per_message", ctypes.c_int32),
        ("messages", ctypes.c_int64),
        ("bytes_sent_per_rank", ctypes.c_int64),
        ("peak_intermediate_slots", ctypes.c_int32),
        ("n_occupancy", ctypes.c_int32),
        ("occupancy_per_round", ctypes.c_int32 * 512),
    ]

    def as_dict(self) -> dict:
        return {
            "rounds": self.rounds,
            "messages": self.messages,
            "max_chunks_per_message": self.max_chunks_per_message,
            "bytes_sent_per_rank": self.bytes_sent_per_rank,
            "peak_intermediate_slots": self.peak_intermediate_slots,
            "occupancy_per_round": list(self.occupancy_per_round[: self.n_occupancy]),
        }


def build() -> None:
    """Compile the C restatement (and the reference, when its sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_lib = None
_ref = None

I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)
VP = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.po_schedule.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, I32P, ctypes.c_int64, I64P]
        L.po_mirror.argtypes = [I32P, ctypes.c_int64, I32P, ctypes.c_int64, I64P]
        L.po_validate.argtypes = [I32P, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
        L.po_run_allgather.argtypes = [I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, VP, VP, ctypes.POINTER(PoStats)]
        L.po_run_reduce_scatter.argtypes = [I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, VP, VP, ctypes.POINTER(PoStats)]
        L.po_oracle_allgather.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, VP, VP]
        L.po_oracle_reduce_scatter.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, VP, VP]
        L.po_tree_fold.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, VP, VP]
        L.po_random_payload.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, VP]
        L.po_random_payload.restype = None
        L.po_mt19937_64.argtypes = [ctypes.c_uint64, ctypes.c_int64, VP]
        L.po_mt19937_64.restype = None
        L.po_fold.argtypes = [ctypes.c_int, ctypes.c_int, VP, VP, ctypes.c_int64]
        L.po_trace_csv.argtypes = [I32P, ctypes.c_int64, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64]
        L.po_trace_csv.restype = ctypes.c_int64
        L.po_max_trees.argtypes = [ctypes.c_int]
        L.po_pat_buffer_slots.argtypes = [ctypes.c_int, ctypes.c_int]
        L.po_trees_from_buffer.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.po_round_count_formula.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.po_sendable_offsets.argtypes = [ctypes.c_int, ctypes.c_int, I32P, ctypes.c_int]
        L.po_ceil_log2.argtypes = [ctypes.c_int64]
        L.po_dtype_size.argtypes = [ctypes.c_int]
        L.po_dtype_size.restype = ctypes.c_size_t
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (oracle/_ref). Raises if it was not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        R = ctypes.CDLL(REF_SO)
        R.ref_schedule.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, I32P, ctypes.c_int64, I64P]
        R.ref_mirror.argtypes = [I32P, ctypes.c_int64, I32P, ctypes.c_int64, I64P]
        R.ref_validate.argtypes = [I32P, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
        R.ref_run_allgather.argtypes = [I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, VP, VP, I64P, ctypes.c_int, ctypes.c_int]
        R.ref_run_reduce_scatter.argtypes = [I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, VP, VP, I64P, ctypes.c_int, ctypes.c_int]
        R.ref_random_payload.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, VP]
        R.ref_oracle_reduce_scatter.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, VP, VP]
        R.ref_trace_csv.argtypes = [I32P, ctypes.c_int64, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64]
        R.ref_trace_csv.restype = ctypes.c_int64
        R.ref_trees_from_buffer.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        R.ref_round_count_formula.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        R.ref_oracle_sweep.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, I64P]
        R.ref_last_error.restype = ctypes.c_char_p
        R.ref_prepare.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        R.ref_prepare.restype = ctypes.c_void_p
        R.ref_run_prepared.argtypes = [ctypes.c_void_p, ctypes.c_int]
        R.ref_free_prepared.argtypes = [ctypes.c_void_p]
        R.ref_free_prepared.restype = None
        _ref = R
    return _ref


def _i32(a: np.ndarray):
    return a.ctypes.data_as(I32P)


# ------------------------------------------------------------------ schedules

def schedule(kind: int, algorithm: int, n: int, trees: int = 1) -> np.ndarray:
    cap = 16 + 8 * max(n, 1) * (max(n, 1) + 2)
    buf = np.zeros(cap, np.int32)
    ln = ctypes.c_int64()
    rc = lib().po_schedule(kind, algorithm, n, trees, _i32(buf), cap, ctypes.byref(ln))
    if rc:
        raise OracleError(rc, "po_schedule")
    return buf[: ln.value].copy()


def pat_allgather(n: int, trees: int) -> np.ndarray:
    return schedule(ALLGATHER, PAT, n, trees)


def pat_reduce_scatter(n: int, trees: int) -> np.ndarray:
    return schedule(REDUCESCATTER, PAT, n, trees)


def mirror(s: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(s, np.int32)
    out = np.zeros(len(s) + 16, np.int32)
    ln = ctypes.c_int64()
    rc = lib().po_mirror(_i32(s), len(s), _i32(out), len(out), ctypes.byref(ln))
    if rc:
        raise OracleError(rc, "po_mirror")
    return out[: ln.value].copy()


def validate(s: np.ndarray) -> tuple[int, str]:
    s = np.ascontiguousarray(s, np.int32)
    msg = ctypes.create_string_buffer(4096)
    n = lib().po_validate(_i32(s), len(s), msg, 4096)
    return n, msg.value.decode()


def decode(s) -> dict:
    """Flat int32 encoding -> dict mirroring RelativeSchedule (schedule.hpp:78-86)."""
    s = [int(x) for x in s]
    out = {"kind": s[0], "algorithm": s[1], "n_ranks": s[2],
           "params": {"trees": s[4], "buffer_slots": s[5]} if s[3] else None, "rounds": []}
    p = 7
    for _ in range(s[6]):
        nk = s[p + 5]
        out["rounds"].append({"round": s[p], "dim": s[p + 1], "split": s[p + 2], "peer": s[p + 3],
                              "exchange": bool(s[p + 4]), "chunks": s[p + 6: p + 6 + nk]})
        p += 6 + nk
    return out


def encode(d: dict) -> np.ndarray:
    v = [d["kind"], d["algorithm"], d["n_ranks"], 1 if d.get("params") else 0,
         (d.get("params") or {}).get("trees", 0), (d.get("params") or {}).get("buffer_slots", 0),
         len(d["rounds"])]
    for r in d["rounds"]:
        v += [r["round"], r["dim"], r["split"], r["peer"], int(r["exchange"]), len(r["chunks"])]
        v += list(r["chunks"])
    return np.array(v, np.int32)


def max_trees(n: int) -> int:
    return lib().po_max_trees(n)


def valid_tree_counts(n: int) -> list[int]:
    out, t = [], 1
    while t <= max_trees(n):
        out.append(t)
        t *= 2
    return out


def trees_from_buffer(buffer_bytes: int, chunk_bytes: int, n: int) -> int:
    t = ctypes.c_int()
    rc = lib().po_trees_from_buffer(buffer_bytes, chunk_bytes, n, ctypes.byref(t))
    if rc:
        raise OracleError(rc, "po_trees_from_buffer")
    return t.value


def round_count_formula(n: int, trees: int) -> int:
    t = ctypes.c_int()
    rc = lib().po_round_count_formula(n, trees, ctypes.byref(t))
    if rc:
        raise OracleError(rc, "po_round_count_formula")
    return t.value


def sendable_offsets(n: int, dim: int) -> list[int]:
    out = np.zeros(max(n, 1), np.int32)
    c = lib().po_sendable_offsets(n, dim, _i32(out), len(out))
    return [int(x) for x in out[:c]]


def trace_csv(s: np.ndarray, chunk_bytes: int) -> str:
    s = np.ascontiguousarray(s, np.int32)
    cap = 1 << 20
    buf = ctypes.create_string_buffer(cap)
    ln = lib().po_trace_csv(_i32(s), len(s), chunk_bytes, buf, cap)
    return buf.value.decode()


# ------------------------------------------------------------------ payloads / executors

def random_payload(dtype: int, nchunks: int, elems: int, seed: int) -> np.ndarray:
    out = np.zeros(nchunks * elems, NP_DTYPE[dtype])
    lib().po_random_payload(dtype, nchunks, elems, seed, out.ctypes.data)
    return out


def run_allgather(s: np.ndarray, dtype: int, payload: np.ndarray, elems: int):
    """payload: n*elems (rank-major). Returns (out[n, n*elems], stats dict)."""
    s = np.ascontiguousarray(s, np.int32)
    n = int(s[2])
    payload = np.ascontiguousarray(payload)
    out = np.zeros(n * n * elems, payload.dtype)
    st = PoStats()
    rc = lib().po_run_allgather(_i32(s), len(s), dtype, elems, payload.ctypes.data, out.ctypes.data, ctypes.byref(st))
    if rc:
        raise OracleError(rc, "po_run_allgather")
    return out.reshape(n, n * elems), st.as_dict()


def run_reduce_scatter(s: np.ndarray, dtype: int, op: int, payload: np.ndarray, elems: int):
    """payload: n*n*elems (chunks[s*n+d]). Returns (out[n, elems], stats dict)."""
    s = np.ascontiguousarray(s, np.int32)
    n = int(s[2])
    payload = np.ascontiguousarray(payload)
    out = np.zeros(n * elems, payload.dtype)
    st = PoStats()
    rc = lib().po_run_reduce_scatter(_i32(s), len(s), dtype, op, elems, payload.ctypes.data, out.ctypes.data, ctypes.byref(st))
    if rc:
        raise OracleError(rc, "po_run_reduce_scatter")
    return out.reshape(n, elems), st.as_dict()


def oracle_reduce_scatter(n: int, dtype: int, op: int, payload: np.ndarray, elems: int) -> np.ndarray:
    payload = np.ascontiguousarray(payload)
    out = np.zeros(n * elems, payload.dtype)
    rc = lib().po_oracle_reduce_scatter(n, dtype, op, elems, payload.ctypes.data, out.ctypes.data)
    if rc:
        raise OracleError(rc, "po_oracle_reduce_scatter")
    return out.reshape(n, elems)


def tree_fold(n: int, dtype: int, op: int, column: np.ndarray):
    column = np.ascontiguousarray(column)
    out = np.zeros(1, column.dtype)
    rc = lib().po_tree_fold(n, dtype, op, column.ctypes.data, out.ctypes.data)
    if rc:
        raise OracleError(rc, "po_tree_fold")
    return out[0]


def fold(dtype: int, op: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a).copy()
    b = np.ascontiguousarray(b)
    rc = lib().po_fold(dtype, op, a.ctypes.data, b.ctypes.data, a.size)
    if rc:
        raise OracleError(rc, "po_fold")
    return a

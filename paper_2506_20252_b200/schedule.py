"""Rank-relative schedules, mirroring the reference's schedule/algorithms API.

Reference: /root/reference/proj/include/patsim/schedule.hpp:56-117 and algorithms.hpp:10-62.
Generation, mirroring, validation and slot accounting run in the product's C++ host code
(``csrc/schedule.cpp``) through the C ABI; this module only converts to Python objects.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib


class CollectiveKind(IntEnum):  # schedule.hpp:11
    AllGather = 0
    ReduceScatter = 1


class Algorithm(IntEnum):  # schedule.hpp:13
    Ring = 0
    BruckNearest = 1
    BruckFarthest = 2
    RecursiveDoubling = 3
    Pat = 4


@dataclass
class PatParams:  # schedule.hpp:49-53
    trees: int = 1
    buffer_slots: int = 1


@dataclass
class RelativeRound:  # schedule.hpp:64-76
    round_index: int = 0
    dimension: int = 0
    split_index: int = 0
    peer_send_offset: int = 0
    exchange: bool = False
    chunk_offsets: list = field(default_factory=list)

    def received_offsets(self, n_ranks: int) -> list:  # schedule.cpp:24-32
        if self.exchange:
            return [k ^ abs(self.peer_send_offset) for k in self.chunk_offsets]
        return [(k + self.peer_send_offset) % n_ranks for k in self.chunk_offsets]


@dataclass
class RelativeSchedule:  # schedule.hpp:78-86
    kind: CollectiveKind = CollectiveKind.AllGather
    algorithm: Algorithm = Algorithm.Ring
    n_ranks: int = 1
    params: Optional[PatParams] = None
    rounds: list = field(default_factory=list)

    def encode(self) -> np.ndarray:
        v = [int(self.kind), int(self.algorithm), self.n_ranks, 1 if self.params else 0,
             self.params.trees if self.params else 0, self.params.buffer_slots if self.params else 0,
             len(self.rounds)]
        for r in self.rounds:
            v += [r.round_index, r.dimension, r.split_index, r.peer_send_offset, int(r.exchange),
                  len(r.chunk_offsets)] + list(r.chunk_offsets)
        return np.array(v, np.int32)

    @staticmethod
    def decode(buf) -> "RelativeSchedule":
        b = [int(x) for x in buf]
        s = RelativeSchedule(CollectiveKind(b[0]), Algorithm(b[1]), b[2],
                             PatParams(b[4], b[5]) if b[3] else None, [])
        p = 7
        for _ in range(b[6]):
            nk = b[p + 5]
            s.rounds.append(RelativeRound(b[p], b[p + 1], b[p + 2], b[p + 3], bool(b[p + 4]),
                                          b[p + 6: p + 6 + nk]))
            p += 6 + nk
        return s


def _i32(a: np.ndarray):
    return a.ctypes.data_as(_lib.I32P)


def build(kind: int, algorithm: int, n_ranks: int, trees: int = 1) -> RelativeSchedule:
    cap = 64 + 8 * max(n_ranks, 1) * (max(n_ranks, 1) + 2)
    buf = np.zeros(cap, np.int32)
    ln = ctypes.c_size_t()
    check(lib().patScheduleBuild(int(kind), int(algorithm), n_ranks, trees, _i32(buf), cap, ctypes.byref(ln)),
          "patScheduleBuild")
    return RelativeSchedule.decode(buf[: ln.value])


def pat_allgather(n_ranks: int, trees: int) -> RelativeSchedule:  # algorithms.hpp:54
    return build(CollectiveKind.AllGather, Algorithm.Pat, n_ranks, trees)


def pat_reduce_scatter(n_ranks: int, trees: int) -> RelativeSchedule:  # algorithms.hpp:62
    return build(CollectiveKind.ReduceScatter, Algorithm.Pat, n_ranks, trees)


def ring_allgather(n_ranks: int) -> RelativeSchedule:
    return build(CollectiveKind.AllGather, Algorithm.Ring, n_ranks)


def bruck_nearest(n_ranks: int) -> RelativeSchedule:
    return build(CollectiveKind.AllGather, Algorithm.BruckNearest, n_ranks)


def bruck_farthest(n_ranks: int) -> RelativeSchedule:
    return build(CollectiveKind.AllGather, Algorithm.BruckFarthest, n_ranks)


def recursive_doubling(n_ranks: int) -> RelativeSchedule:
    return build(CollectiveKind.AllGather, Algorithm.RecursiveDoubling, n_ranks)


def mirror_schedule(s: RelativeSchedule) -> RelativeSchedule:  # algorithms.hpp:59
    enc = s.encode()
    out = np.zeros(len(enc) + 16, np.int32)
    ln = ctypes.c_size_t()
    check(lib().patScheduleMirror(_i32(enc), len(enc), _i32(out), len(out), ctypes.byref(ln)), "patScheduleMirror")
    return RelativeSchedule.decode(out[: ln.value])


def validate(s: RelativeSchedule) -> tuple[int, str]:  # schedule.hpp:115
    """Returns (violation count, first message)."""
    enc = s.encode()
    nv = ctypes.c_int()
    msg = ctypes.create_string_buffer(4096)
    check(lib().patScheduleValidate(_i32(enc), len(enc), ctypes.byref(nv), msg, 4096), "patScheduleValidate")
    return nv.value, msg.value.decode()


def stats(s: RelativeSchedule, chunk_bytes: int) -> dict:
    """ExecStats (simulate.hpp:43-53) from the schedule alone."""
    enc = s.encode()
    st = _lib.ExecStats()
    check(lib().patScheduleStats(_i32(enc), len(enc), chunk_bytes, ctypes.byref(st)), "patScheduleStats")
    return {"rounds": st.rounds, "messages": st.messages, "max_chunks_per_message": st.max_chunks_per_message,
            "bytes_sent_per_rank": st.bytes_sent_per_rank, "peak_intermediate_slots": st.peak_intermediate_slots,
            "occupancy_per_round": list(st.occupancy_per_round[: st.n_occupancy])}


def trace_csv(s: RelativeSchedule, chunk_bytes: int) -> str:  # simulate.hpp:98-100
    enc = s.encode()
    ln = ctypes.c_size_t()
    lib().patScheduleTraceCsv(_i32(enc), len(enc), chunk_bytes, None, 0, ctypes.byref(ln))
    buf = ctypes.create_string_buffer(ln.value + 1)
    check(lib().patScheduleTraceCsv(_i32(enc), len(enc), chunk_bytes, buf, ln.value + 1, ctypes.byref(ln)),
          "patScheduleTraceCsv")
    return buf.value.decode()


def max_trees(n_ranks: int) -> int:  # algorithms.hpp:12
    t = ctypes.c_int()
    check(lib().patMaxTrees(n_ranks, ctypes.byref(t)), "patMaxTrees")
    return t.value


def valid_tree_counts(n_ranks: int) -> list:  # algorithms.hpp:15
    out, t = [], 1
    while t <= max_trees(n_ranks):
        out.append(t)
        t *= 2
    return out


def trees_from_buffer(buffer_bytes: int, chunk_bytes: int, n_ranks: int) -> int:  # algorithms.hpp:21
    t = ctypes.c_int()
    check(lib().patTreesFromBuffer(buffer_bytes, chunk_bytes, n_ranks, ctypes.byref(t)), "patTreesFromBuffer")
    return t.value


def pat_buffer_slots(n_ranks: int, trees: int) -> int:  # algorithms.hpp:24
    t = ctypes.c_int()
    check(lib().patPatBufferSlots(n_ranks, trees, ctypes.byref(t)), "patPatBufferSlots")
    return t.value


def round_count_formula(n_ranks: int, trees: int) -> int:  # algorithms.hpp:28
    t = ctypes.c_int()
    check(lib().patRoundCountFormula(n_ranks, trees, ctypes.byref(t)), "patRoundCountFormula")
    return t.value

"""Rank-relative schedules, mirroring the reference's schedule/algorithms API.

Reference: /root/reference/proj/include/patsim/schedule.hpp:56-117 and algorithms.hpp:10-62.
Generation, mirroring, validation and slot accounting run in the product's C++ host code
(``csrc/schedule.cpp``) through the C ABI; this module only converts to Python objects.
"""
from __future__ import annotations

import ctypes
import json
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


# ------------------------------------------------------------------ schedule files
# The reference's schedule JSON format (serialize.cpp:49-101, proj/README.md:95-112): what
# `patsim schedule` writes and `patsim verify` reads. Imported schedules reach the GPU executor
# through patAllGatherSchedule / patReduceScatterSchedule, which validate them first.

_ALGO_TAGS = {Algorithm.Ring: "ring", Algorithm.BruckNearest: "bruck-nearest",
              Algorithm.BruckFarthest: "bruck-farthest", Algorithm.RecursiveDoubling: "recursive-doubling",
              Algorithm.Pat: "pat"}
_KIND_TAGS = {CollectiveKind.AllGather: "allgather", CollectiveKind.ReduceScatter: "reducescatter"}


class ParseError(RuntimeError):  # serialize.hpp:12
    pass


def schedule_to_json(s: RelativeSchedule, indent: int = 2) -> str:
    """serialize.cpp:49-72: key order algorithm, kind, n_ranks, params, rounds; arrays of
    offsets on one line; the text nlohmann::ordered_json::dump(indent) produces, plus a newline."""
    params = {} if s.params is None else {"trees": s.params.trees, "buffer_slots": s.params.buffer_slots}
    rounds = [{"round": r.round_index, "dim": r.dimension, "split": r.split_index, "peer": r.peer_send_offset,
               "chunks": list(r.chunk_offsets)} for r in s.rounds]
    if indent < 0:
        doc = {"algorithm": _ALGO_TAGS[Algorithm(s.algorithm)], "kind": _KIND_TAGS[CollectiveKind(s.kind)],
               "n_ranks": s.n_ranks, "params": params, "rounds": rounds}
        return json.dumps(doc, separators=(",", ":")) + "\n"
    pad = " " * indent

    def obj(d: dict, level: int) -> str:
        if not d:
            return "{}"
        inner = pad * (level + 1)
        items = []
        for k, v in d.items():
            if isinstance(v, list) and (not v or not isinstance(v[0], dict)):
                val = "[" + ",".join(str(x) for x in v) + "]"
            elif isinstance(v, list):
                val = "[\n" + ",\n".join(inner + pad + obj(x, level + 2) for x in v) + "\n" + inner + "]"
            elif isinstance(v, dict):
                val = obj(v, level + 1)
            else:
                val = json.dumps(v)
            items.append(f"{inner}{json.dumps(k)}: {val}")
        return "{\n" + ",\n".join(items) + "\n" + pad * level + "}"

    doc = {"algorithm": _ALGO_TAGS[Algorithm(s.algorithm)], "kind": _KIND_TAGS[CollectiveKind(s.kind)],
           "n_ranks": s.n_ranks, "params": params, "rounds": rounds}
    return obj(doc, 0) + "\n"


def schedule_from_json(text: str) -> RelativeSchedule:
    """serialize.cpp:74-101, with the reference's ParseError messages."""
    try:
        doc = json.loads(text)
    except (ValueError, TypeError):
        raise ParseError("malformed JSON in schedule") from None

    def field(o: dict, name: str, where: str, types):
        if not isinstance(o, dict) or name not in o:
            raise ParseError(f'{where} is missing field "{name}"')
        v = o[name]
        if not isinstance(v, types) or (isinstance(v, bool) and types is not bool):
            raise ParseError(f'{where} field "{name}" has the wrong type')
        return v

    algo = {v: k for k, v in _ALGO_TAGS.items()}
    kind = {v: k for k, v in _KIND_TAGS.items()}
    atag = field(doc, "algorithm", "schedule", str)
    if atag not in algo:
        raise ParseError(f'unknown algorithm tag "{atag}"')
    ktag = field(doc, "kind", "schedule", str)
    if ktag not in kind:
        raise ParseError(f'unknown kind "{ktag}"')
    n = field(doc, "n_ranks", "schedule", int)
    if "params" not in doc:
        raise ParseError('schedule is missing field "params"')
    params = doc["params"]
    if not isinstance(params, dict):
        raise ParseError('schedule field "params" must be an object')
    pp = None
    if params:
        pp = PatParams(field(params, "trees", "params", int), field(params, "buffer_slots", "params", int))
    if "rounds" not in doc:
        raise ParseError('schedule is missing field "rounds"')
    rounds = doc["rounds"]
    if not isinstance(rounds, list):
        raise ParseError('schedule field "rounds" must be an array')
    exchange = algo[atag] == Algorithm.RecursiveDoubling  # XOR partnering implied by the algorithm
    out = RelativeSchedule(kind[ktag], algo[atag], n, pp, [])
    for r in rounds:
        rr = RelativeRound(field(r, "round", "round", int), field(r, "dim", "round", int),
                           field(r, "split", "round", int), field(r, "peer", "round", int), exchange, [])
        chunks = field(r, "chunks", "round", list)
        if any(not isinstance(x, int) or isinstance(x, bool) for x in chunks):
            raise ParseError('round field "chunks" has the wrong type')
        rr.chunk_offsets = list(chunks)
        out.rounds.append(rr)
    return out


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

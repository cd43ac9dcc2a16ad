"""CPU tests of the product's host side through the C ABI (no GPU needed).

* libpatb200.so loads and exports every function include/pat_b200.h declares;
* the product's own C++ schedule generator / mirror / validate / slot accounting / trace
  match the reference-generated golden fixtures (tests/golden) and the reference's unit-test
  constants — the same bar the oracle is held to;
* error codes map the reference's exception classes.
"""
import json
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2506_20252_b200 import _lib, schedule as S
from paper_2506_20252_b200.schedule import CollectiveKind, RelativeSchedule

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "pat_b200.h")).read()
    declared = set(re.findall(r"^(?:patResult_t|const char\*)\s+(pat\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.SYMBOLS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    v = __import__("ctypes").c_int()
    assert L.patGetVersion(__import__("ctypes").byref(v)) == 0 and v.value == 10000
    assert L.patGetErrorString(33) == b"InvalidScheduleError"


def test_python_constants_match_header_enums():
    """The binding's protocol / op / dtype numbers are the header's (ABI drift guard)."""
    header = open(os.path.join(ROOT, "include", "pat_b200.h")).read()
    enum = {k: int(v) for k, v in re.findall(r"\b(pat\w+)\s*=\s*(\d+)", header)}
    assert {k: enum[k] for k in ("patProtoAuto", "patProtoLL", "patProtoSimple", "patProtoPull", "patProtoLL32")} == {
        "patProtoAuto": _lib.PROTO_AUTO, "patProtoLL": _lib.PROTO_LL, "patProtoSimple": _lib.PROTO_SIMPLE,
        "patProtoPull": _lib.PROTO_PULL, "patProtoLL32": _lib.PROTO_LL32}
    assert [enum[k] for k in ("patSum", "patProd", "patMax", "patMin")] == [_lib.SUM, _lib.PROD, _lib.MAX, _lib.MIN]
    names = ["patInt8", "patUint8", "patInt32", "patUint32", "patInt64", "patUint64", "patFloat16", "patFloat32",
             "patFloat64", "patBfloat16"]
    consts = [_lib.INT8, _lib.UINT8, _lib.INT32, _lib.UINT32, _lib.INT64, _lib.UINT64, _lib.FLOAT16, _lib.FLOAT32,
              _lib.FLOAT64, _lib.BFLOAT16]
    assert [enum[k] for k in names] == consts


def test_library_has_sm100a_code():
    so = _lib.LIB_PATH
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.fixture(scope="module")
def golden(golden_dir):
    with open(os.path.join(golden_dir, "schedules.json")) as f:
        return json.load(f)


def test_schedules_match_reference(golden):
    for case in golden["schedules"]:
        want = case["schedule"]
        if isinstance(want, dict):
            with pytest.raises(_lib.PatError) as ei:
                S.build(case["kind"], case["algorithm"], case["n"], case["trees"] or 1)
            assert ei.value.kind == want["error"]
            continue
        got = S.build(case["kind"], case["algorithm"], case["n"], case["trees"] or 1)
        assert [int(x) for x in got.encode()] == want, (case["kind"], case["algorithm"], case["n"], case["trees"])


def test_schedule_errors(golden):
    for case in golden["errors"]:
        algo = S.Algorithm.RecursiveDoubling if case.get("algorithm") == "recursive-doubling" else S.Algorithm.Pat
        with pytest.raises(_lib.PatError) as ei:
            S.build(0, algo, case["n"], case.get("trees", 1))
        assert ei.value.kind == case["result"]["error"]


def test_validate_messages_match_reference(golden_dir):
    misc = json.load(open(os.path.join(golden_dir, "misc.json")))
    for name, case in misc["validate"].items():
        s = RelativeSchedule.decode(case["schedule"])
        nv, first = S.validate(s)
        assert (nv, first) == (case["violations"], case["first"]), name
    assert S.trace_csv(S.pat_allgather(4, 1), 8) == misc["trace_pat_4_1_8"]
    assert S.trace_csv(S.pat_allgather(8, 4), 1 << 20) == misc["trace_pat_8_4_1MiB"]
    for c in misc["trees_from_buffer"]:
        if c["rc"] == 0:
            assert S.trees_from_buffer(c["buffer"], c["chunk"], c["n"]) == c["trees"]
        else:
            with pytest.raises(_lib.PatError):
                S.trees_from_buffer(c["buffer"], c["chunk"], c["n"])
    for c in misc["round_count_formula"]:
        if c["rc"] == 0:
            assert S.round_count_formula(c["n"], c["trees"]) == c["rounds"]
        else:
            with pytest.raises(_lib.PatError) as ei:
                S.round_count_formula(c["n"], c["trees"])


def test_stats_match_reference_executor(golden_dir):
    ex = np.load(os.path.join(golden_dir, "executor.npz"))
    for key in ex["index"]:
        n, t, seed, dt = (int(x[1:]) for x in str(key).split("_"))
        if seed or dt != O.INT64:
            continue
        st = S.stats(S.pat_allgather(n, t), 4 * 8)
        ref = [int(x) for x in ex[f"ag_stats_{key}"]]
        assert [st["rounds"], st["messages"], st["max_chunks_per_message"], st["bytes_sent_per_rank"],
                st["peak_intermediate_slots"], len(st["occupancy_per_round"])] + st["occupancy_per_round"] == ref
        st = S.stats(S.pat_reduce_scatter(n, t), 4 * 8)
        assert st["occupancy_per_round"] == [int(x) for x in ex[f"rs_stats_{key}"][6:]]


def test_reference_unit_constants():
    # test_algorithms.cpp:143-155, 245-255; test_simulate.cpp:57-99
    s = S.pat_allgather(8, 2)
    assert [r.chunk_offsets for r in s.rounds] == [[0], [4, 0], [6, 4], [2, 0]]
    assert s.params.trees == 2 and s.params.buffer_slots == 4
    m = S.mirror_schedule(s)
    assert m.kind == CollectiveKind.ReduceScatter
    assert [r.chunk_offsets for r in m.rounds] == [[3, 1], [7, 5], [6, 2], [4]]
    assert S.mirror_schedule(m) == s
    assert S.stats(s, 16)["occupancy_per_round"] == [1, 3, 1, 0]
    assert S.stats(S.pat_allgather(8, 1), 8)["peak_intermediate_slots"] == 2
    assert S.stats(S.pat_allgather(16, 4), 8)["occupancy_per_round"] == [1, 3, 7, 3, 0]
    assert S.valid_tree_counts(8) == [1, 2, 4] and S.max_trees(16) == 8
    r = s.rounds[1]
    assert r.received_offsets(8) == [6, 2]
    # acceptance criterion 6: peak <= ceil(log2 n) for n <= 8, every T
    for n in range(2, 9):
        for t in S.valid_tree_counts(n):
            assert S.stats(S.pat_allgather(n, t), 1)["peak_intermediate_slots"] <= O.lib().po_ceil_log2(n)


def test_comm_init_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.PatError):
        from paper_2506_20252_b200 import PatComm
        PatComm.init_all(2, [0, 0])


def test_group_calls_without_gpu():
    """patGroupEnd without patGroupStart is InvalidUsage; nested groups balance (no GPU needed)."""
    from paper_2506_20252_b200 import _lib as L
    lib = L.lib()
    assert lib.patGroupEnd() == 5
    assert lib.patGroupStart() == 0 and lib.patGroupStart() == 0
    assert lib.patGroupEnd() == 0 and lib.patGroupEnd() == 0
    assert lib.patGroupEnd() == 5

"""Pin the CPU oracle (oracle/pat_oracle.c) to the reference.

Two sources of truth, both from the reference itself:
  * tests/golden/*  — fixtures produced by the compiled reference (make_golden.py);
  * the known-answer constants of the reference's own unit tests, cited file:line
    (proj/tests/test_algorithms.cpp, test_simulate.cpp, test_schedule.cpp).
"""
import json
import os

import numpy as np
import pytest

import oracle as O


@pytest.fixture(scope="module")
def schedules(golden_dir):
    with open(os.path.join(golden_dir, "schedules.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def executor(golden_dir):
    return np.load(os.path.join(golden_dir, "executor.npz"))


@pytest.fixture(scope="module")
def misc(golden_dir):
    with open(os.path.join(golden_dir, "misc.json")) as f:
        return json.load(f)


def chunk_sets(s):
    return [r["chunks"] for r in O.decode(s)["rounds"]]


def dims(s):
    return [r["dim"] for r in O.decode(s)["rounds"]]


# ------------------------------------------------------------------ golden fixtures

def test_every_reference_schedule_matches(schedules):
    for case in schedules["schedules"]:
        want = case["schedule"]
        if isinstance(want, dict):  # reference threw (recursive doubling on non-power-of-two n)
            with pytest.raises(O.OracleError) as ei:
                O.schedule(case["kind"], case["algorithm"], case["n"], case["trees"] or 1)
            assert ei.value.kind == want["error"]
            continue
        got = O.schedule(case["kind"], case["algorithm"], case["n"], case["trees"] or 1)
        assert [int(x) for x in got] == want, (case["kind"], case["algorithm"], case["n"], case["trees"])


def test_reference_schedule_errors(schedules):
    for case in schedules["errors"]:
        algo = O.RECURSIVE_DOUBLING if case.get("algorithm") == "recursive-doubling" else O.PAT
        with pytest.raises(O.OracleError) as ei:
            O.schedule(O.ALLGATHER, algo, case["n"], case.get("trees", 1))
        assert ei.value.kind == case["result"]["error"]


def test_executor_outputs_and_stats_bit_exact(executor):
    for key in executor["index"]:
        n, t, seed, dt = (int(x[1:]) for x in str(key).split("_"))
        elems = 4
        ag = O.pat_allgather(n, t)
        rs = O.pat_reduce_scatter(n, t)
        p = executor[f"ag_in_{key}"]
        assert np.array_equal(O.random_payload(dt, n, elems, seed).view(np.uint64), p.view(np.uint64))
        out, st = O.run_allgather(ag, dt, p, elems)
        assert np.array_equal(out.reshape(-1).view(np.uint64), executor[f"ag_out_{key}"].view(np.uint64)), key
        ref_st = executor[f"ag_stats_{key}"]
        assert [st["rounds"], st["messages"], st["max_chunks_per_message"], st["bytes_sent_per_rank"],
                st["peak_intermediate_slots"], len(st["occupancy_per_round"])] + st["occupancy_per_round"] \
            == [int(x) for x in ref_st], key
        p = executor[f"rs_in_{key}"]
        assert np.array_equal(O.random_payload(dt, n * n, elems, seed).view(np.uint64), p.view(np.uint64))
        out, st = O.run_reduce_scatter(rs, dt, O.SUM, p, elems)
        # bit-exact, floats included: the restatement reproduces the PAT tree order
        assert np.array_equal(out.reshape(-1).view(np.uint64), executor[f"rs_out_{key}"].view(np.uint64)), key
        ref_st = executor[f"rs_stats_{key}"]
        assert st["occupancy_per_round"] == [int(x) for x in ref_st[6:]], key
        ro = O.oracle_reduce_scatter(n, dt, O.SUM, p, elems)
        assert np.array_equal(ro.reshape(-1).view(np.uint64), executor[f"rs_rankorder_{key}"].view(np.uint64))


def test_closed_form_tree_matches_reference_float_order(executor):
    """out[r] = tree over x_j = chunks[(r+j)%n][r]; T-independent."""
    for key in executor["index"]:
        n, t, seed, dt = (int(x[1:]) for x in str(key).split("_"))
        if dt != O.FLOAT64 or n > 8:
            continue
        p = executor[f"rs_in_{key}"].reshape(n, n, 4)
        want = executor[f"rs_out_{key}"].reshape(n, 4)
        for r in range(n):
            for e in range(4):
                col = np.array([p[(r + j) % n, r, e] for j in range(n)])
                assert O.tree_fold(n, O.FLOAT64, O.SUM, col) == want[r, e]


def test_validate_messages(misc):
    for name, case in misc["validate"].items():
        nv, first = O.validate(np.array(case["schedule"], np.int32))
        assert nv == case["violations"], name
        assert first == case["first"], name


def test_trace_csv(misc):
    assert O.trace_csv(O.pat_allgather(4, 1), 8) == misc["trace_pat_4_1_8"]
    assert O.trace_csv(O.pat_allgather(8, 4), 1 << 20) == misc["trace_pat_8_4_1MiB"]


def test_trees_from_buffer_and_formula(misc):
    for c in misc["trees_from_buffer"]:
        if c["rc"] == 0:
            assert O.trees_from_buffer(c["buffer"], c["chunk"], c["n"]) == c["trees"]
        else:
            with pytest.raises(O.OracleError):
                O.trees_from_buffer(c["buffer"], c["chunk"], c["n"])
    for c in misc["round_count_formula"]:
        if c["rc"] == 0:
            assert O.round_count_formula(c["n"], c["trees"]) == c["rounds"]
        else:
            with pytest.raises(O.OracleError):
                O.round_count_formula(c["n"], c["trees"])
    assert misc["reference_oracle_sweep_1_64_mismatches"] == 0


# ------------------------------------------------------------------ reference unit-test constants

def test_pat_8_2_known_answer():  # test_algorithms.cpp:143-155
    s = O.pat_allgather(8, 2)
    assert chunk_sets(s) == [[0], [4, 0], [6, 4], [2, 0]]
    assert dims(s) == [2, 1, 0, 0]
    d = O.decode(s)
    assert [r["split"] for r in d["rounds"]][2:] == [0, 1]
    assert d["params"] == {"trees": 2, "buffer_slots": 4}


def test_pat_16_known_answers():  # test_algorithms.cpp:173-192
    assert chunk_sets(O.pat_allgather(16, 4)) == [[0], [8, 0], [12, 8, 4, 0], [14, 12, 10, 8], [6, 4, 2, 0]]
    assert dims(O.pat_allgather(16, 4)) == [3, 2, 1, 0, 0]
    got = [(r["dim"], r["chunks"][0]) for r in O.decode(O.pat_allgather(16, 1))["rounds"]]
    assert got == [(3, 0), (2, 8), (1, 12), (0, 14), (0, 12), (1, 8), (0, 10), (0, 8),
                   (2, 0), (1, 4), (0, 6), (0, 4), (1, 0), (0, 2), (0, 0)]


def test_full_aggregation_is_bruck_farthest():  # test_algorithms.cpp:157-162
    for n in range(2, 257):
        a = O.decode(O.pat_allgather(n, O.max_trees(n)))["rounds"]
        b = O.decode(O.schedule(O.ALLGATHER, O.BRUCK_FARTHEST, n))["rounds"]
        assert a == b


def test_mirror_known_answer_and_involution():  # test_algorithms.cpp:245-268
    m = O.mirror(O.pat_allgather(8, 2))
    d = O.decode(m)
    assert d["kind"] == O.REDUCESCATTER
    assert chunk_sets(m) == [[3, 1], [7, 5], [6, 2], [4]]
    assert dims(m) == [0, 0, 1, 2]
    assert d["rounds"][0]["peer"] == -1
    assert [r["split"] for r in d["rounds"]][:2] == [0, 1]
    for n in (1, 2, 3, 5, 8, 16, 31, 64):
        for t in O.valid_tree_counts(n):
            s = O.pat_allgather(n, t)
            assert np.array_equal(O.mirror(O.mirror(s)), s)
    assert dims(O.pat_reduce_scatter(16, 4)) == [0, 0, 1, 2, 3]


def test_sendable_offsets():  # test_algorithms.cpp:298-304
    assert O.sendable_offsets(8, 2) == [0]
    assert O.sendable_offsets(8, 0) == [6, 4, 2, 0]
    assert O.sendable_offsets(7, 0) == [4, 2, 0]
    assert O.sendable_offsets(7, 1) == [4, 0]
    assert O.sendable_offsets(3, 0) == [0]


def test_occupancy_traces():  # test_simulate.cpp:57-99
    ones = lambda n, e: np.ones(n * e, np.int64)
    _, st = O.run_allgather(O.pat_allgather(8, 2), O.INT64, ones(8, 2), 2)
    assert st["occupancy_per_round"] == [1, 3, 1, 0] and st["peak_intermediate_slots"] == 3
    _, st = O.run_allgather(O.pat_allgather(8, 1), O.INT64, ones(8, 1), 1)
    assert st["peak_intermediate_slots"] == 2
    _, st = O.run_allgather(O.pat_allgather(16, 1), O.INT64, ones(16, 1), 1)
    assert st["peak_intermediate_slots"] == 3
    for e in (1, 7, 32):
        _, st = O.run_allgather(O.pat_allgather(16, 4), O.INT64, ones(16, e), e)
        assert st["occupancy_per_round"] == [1, 3, 7, 3, 0]


def test_small_reduce_scatter_known_answers():  # test_simulate.cpp:152-192
    p = np.array([1, 2, 3, 4], np.int64)
    out, _ = O.run_reduce_scatter(O.pat_reduce_scatter(2, 1), O.INT64, O.SUM, p, 1)
    assert out.tolist() == [[4], [6]]
    out, _ = O.run_reduce_scatter(O.pat_reduce_scatter(8, 4), O.INT64, O.SUM, np.ones(64 * 4, np.int64), 4)
    assert (out == 8).all()
    p = np.array([0x7FFFFFFFFFFFFFFF, -1] * 16, np.int64)
    out, _ = O.run_reduce_scatter(O.pat_reduce_scatter(4, 2), O.INT64, O.SUM, p, 2)
    assert np.array_equal(out, O.oracle_reduce_scatter(4, O.INT64, O.SUM, p, 2))


def test_errors_are_typed():  # test_simulate.cpp:194-227
    s = O.pat_allgather(8, 2)
    with pytest.raises(O.OracleError) as ei:
        O.run_allgather(O.pat_reduce_scatter(8, 2), O.INT64, np.zeros(16, np.int64), 2)
    assert ei.value.kind == "SimulationError"
    d = O.decode(s)
    d["rounds"][0]["chunks"] = [5]
    with pytest.raises(O.OracleError) as ei:
        O.run_allgather(O.encode(d), O.INT64, np.zeros(16, np.int64), 2)
    assert ei.value.kind == "InvalidScheduleError"
    with pytest.raises(O.OracleError) as ei:
        O.run_reduce_scatter(O.pat_reduce_scatter(4, 2), O.INT64, 7, np.zeros(32, np.int64), 2)
    assert ei.value.kind == "UnsupportedOpError"


# ------------------------------------------------------------------ extended dtypes (unpinned by reference tests)

@pytest.mark.parametrize("dt", [O.FLOAT32, O.BFLOAT16, O.FLOAT16, O.INT32, O.UINT8, O.INT8, O.UINT32, O.UINT64])
def test_extended_dtype_tree_order(dt):
    """For dtypes the reference lacks, the executor must follow the same T-independent
    tree with per-hop rounding in the wire dtype."""
    elems = 16
    for n in range(2, 9):
        p = O.random_payload(dt, n * n, elems, 5)
        outs = []
        for t in O.valid_tree_counts(n):
            out, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, t), dt, O.SUM, p, elems)
            outs.append(out)
        for o in outs[1:]:
            assert np.array_equal(o, outs[0])
        pp = p.reshape(n, n, elems)
        for r in range(n):
            for e in range(0, elems, 5):
                col = np.array([pp[(r + j) % n, r, e] for j in range(n)])
                assert O.tree_fold(n, dt, O.SUM, col) == outs[0][r, e]


def test_bf16_fp16_rounding_rules():
    bf = lambda x: np.array([x], np.float32).view(np.uint32).astype(np.uint64) >> 16
    # 1 + 2^-8 is a bf16 tie -> rounds to even (1.0); 1 + 3*2^-9 -> up
    one = np.array([0x3F80], np.uint16)
    tiny = np.array([0x3B80], np.uint16)  # 2^-8
    assert O.fold(O.BFLOAT16, O.SUM, one, tiny)[0] == 0x3F80
    h_one = np.array([0x3C00], np.uint16)
    h_half_ulp = np.array([0x1000], np.uint16)  # 2^-11
    assert O.fold(O.FLOAT16, O.SUM, h_one, h_half_ulp)[0] == 0x3C00
    # fp16 subnormal + subnormal stays exact
    a = np.array([0x0001], np.uint16)
    assert O.fold(O.FLOAT16, O.SUM, a, a)[0] == 0x0002
    # overflow to inf
    big = np.array([0x7BFF], np.uint16)
    assert O.fold(O.FLOAT16, O.SUM, big, big)[0] == 0x7C00
    del bf


def test_max_min_prod():
    a = np.array([1.0, -2.0, 3.0], np.float32)
    b = np.array([0.5, 4.0, 3.0], np.float32)
    assert O.fold(O.FLOAT32, O.MAX, a, b).tolist() == [1.0, 4.0, 3.0]
    assert O.fold(O.FLOAT32, O.MIN, a, b).tolist() == [0.5, -2.0, 3.0]
    assert O.fold(O.FLOAT32, O.PROD, a, b).tolist() == [0.5, -8.0, 9.0]
    x = np.array([-1, 5], np.int32)
    y = np.array([2, -7], np.int32)
    assert O.fold(O.INT32, O.MAX, x, y).tolist() == [2, 5]
    ux = x.view(np.uint32)
    uy = y.view(np.uint32)
    assert O.fold(O.UINT32, O.MAX, ux, uy).tolist() == [0xFFFFFFFF, 0xFFFFFFF9]


def test_mt19937_64_reference_value():
    # C++ standard [rand.predef]: the 10000th draw of a default-seeded mt19937_64
    out = np.zeros(10000, np.uint64)
    O.lib().po_mt19937_64(5489, 10000, out.ctypes.data)
    assert int(out[-1]) == 9981545732273789042

"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref/libpatsim_ref.so).

Run in the build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/schedules.json   flat-encoded schedules from the reference generators
                                (algorithms.cpp:105-249) for every (kind, algorithm, n, T)
  tests/golden/executor.npz     run_allgather / run_reduce_scatter outputs + ExecStats on
                                the reference's own seeded payloads (oracle.cpp:92-112),
                                int64 and float64, n = 1..12, every valid T, seeds {0,1,2}
  tests/golden/misc.json        validate() messages on tampered schedules, trace CSV,
                                trees_from_buffer / round_count_formula answers, the
                                reference oracle_sweep result (acceptance criterion 1)
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_schedule(kind, algo, n, t):
    R = O.ref()
    cap = 64 + 8 * n * (n + 2)
    buf = np.zeros(cap, np.int32)
    ln = ctypes.c_int64()
    rc = R.ref_schedule(kind, algo, n, t, buf.ctypes.data_as(O.I32P), cap, ctypes.byref(ln))
    if rc:
        return {"error": O.ERRORS.get(rc, rc), "message": R.ref_last_error().decode()}
    return [int(x) for x in buf[: ln.value]]


def ref_validate(enc):
    R = O.ref()
    s = np.array(enc, np.int32)
    msg = ctypes.create_string_buffer(4096)
    rc = R.ref_validate(s.ctypes.data_as(O.I32P), len(s), msg, 4096)
    return {"violations": -rc, "first": msg.value.decode()}


def tampered():
    """The negative controls of test_schedule.cpp:122-192 / test_simulate.cpp:215-227."""
    cases = {}
    base = O.decode(ref_schedule(0, O.BRUCK_NEAREST, 8, 1))

    def mod(name, fn, src=None):
        d = json.loads(json.dumps(src or base))
        fn(d)
        cases[name] = {"schedule": [int(x) for x in O.encode(d)], **ref_validate(list(O.encode(d)))}

    mod("unheld_offset", lambda d: d["rounds"][0].__setitem__("chunks", [5]))
    mod("coverage_gap", lambda d: d["rounds"].pop())
    mod("duplicate_offset", lambda d: d["rounds"][2].__setitem__("chunks", [0, 1, 1, 2]))
    mod("peer_mismatch", lambda d: d["rounds"][1].__setitem__("peer", 3))
    mod("round_index", lambda d: d["rounds"][1].__setitem__("round", 5))
    mod("offset_range", lambda d: d["rounds"][0].__setitem__("chunks", [0, 9]))

    def selfloop(d):
        d["rounds"][2]["dim"] = 3
        d["rounds"][2]["peer"] = 8
    mod("self_loop", selfloop)
    mod("empty_round", lambda d: d["rounds"][0].__setitem__("chunks", []))
    rs = O.decode(ref_schedule(1, O.PAT, 8, 2))
    mod("rs_forward_twice", lambda d: d["rounds"][2].__setitem__("chunks", [3, 2]), rs)
    mod("rs_lost_offset", lambda d: d["rounds"][3].__setitem__("chunks", [2]), rs)
    mod("rs_own_destination", lambda d: d["rounds"][0].__setitem__("chunks", [3, 0]), rs)
    pat = O.decode(ref_schedule(0, O.PAT, 8, 2))
    mod("pat_unheld", lambda d: d["rounds"][0].__setitem__("chunks", [5]), pat)
    return cases


def main():
    R = O.ref()
    # ---------------- schedules
    scheds = []
    ns = list(range(1, 33)) + [48, 64, 100, 128]
    for n in ns:
        for kind in (O.ALLGATHER, O.REDUCESCATTER):
            for algo in range(5):
                if algo != O.PAT and n > 32:
                    continue
                trees = O.valid_tree_counts(n) if algo == O.PAT else [0]
                for t in trees:
                    scheds.append({"kind": kind, "algorithm": algo, "n": n, "trees": t,
                                   "schedule": ref_schedule(kind, algo, n, t)})
    # invalid tree counts / non-power-of-two errors
    errors = []
    for n, t in [(16, 3), (16, 0), (16, 16), (8, -2), (3, 4)]:
        errors.append({"n": n, "trees": t, "result": ref_schedule(0, O.PAT, n, t)})
    errors.append({"n": 6, "algorithm": "recursive-doubling", "result": ref_schedule(0, O.RECURSIVE_DOUBLING, 6, 0)})
    with open(os.path.join(OUT, "schedules.json"), "w") as f:
        json.dump({"generator": "oracle/_ref/libpatsim_ref.so (reference algorithms.cpp)",
                   "schedules": scheds, "errors": errors}, f, separators=(",", ":"))

    # ---------------- executor
    arrays = {}
    index = []
    elems = 4
    for n in range(1, 13):
        for t in O.valid_tree_counts(n):
            ag = np.array(ref_schedule(0, O.PAT, n, t), np.int32)
            rs = np.array(ref_schedule(1, O.PAT, n, t), np.int32)
            for seed in (0, 1, 2):
                for dt, npdt in ((O.INT64, np.int64), (O.FLOAT64, np.float64)):
                    key = f"n{n}_t{t}_s{seed}_d{dt}"
                    p = np.zeros(n * elems, npdt)
                    R.ref_random_payload(0, dt, n, elems, seed, p.ctypes.data)
                    out = np.zeros(n * n * elems, npdt)
                    st = np.zeros(600, np.int64)
                    rc = R.ref_run_allgather(ag.ctypes.data_as(O.I32P), len(ag), dt, elems, p.ctypes.data,
                                             out.ctypes.data, st.ctypes.data_as(O.I64P), 0, 0)
                    assert rc == 0
                    arrays[f"ag_in_{key}"] = p
                    arrays[f"ag_out_{key}"] = out
                    arrays[f"ag_stats_{key}"] = st[: 6 + st[5]].copy()
                    p = np.zeros(n * n * elems, npdt)
                    R.ref_random_payload(1, dt, n, elems, seed, p.ctypes.data)
                    out = np.zeros(n * elems, npdt)
                    rc = R.ref_run_reduce_scatter(rs.ctypes.data_as(O.I32P), len(rs), dt, elems, p.ctypes.data,
                                                  out.ctypes.data, st.ctypes.data_as(O.I64P), 0, 0)
                    assert rc == 0
                    arrays[f"rs_in_{key}"] = p
                    arrays[f"rs_out_{key}"] = out
                    arrays[f"rs_stats_{key}"] = st[: 6 + st[5]].copy()
                    ro = np.zeros(n * elems, npdt)
                    R.ref_oracle_reduce_scatter(dt, n, elems, p.ctypes.data, ro.ctypes.data)
                    arrays[f"rs_rankorder_{key}"] = ro
                    index.append(key)
    arrays["index"] = np.array(index)
    np.savez_compressed(os.path.join(OUT, "executor.npz"), **arrays)

    # ---------------- misc
    misc = {"validate": tampered()}
    s = np.array(ref_schedule(0, O.PAT, 4, 1), np.int32)
    buf = ctypes.create_string_buffer(1 << 16)
    R.ref_trace_csv(s.ctypes.data_as(O.I32P), len(s), 8, buf, 1 << 16)
    misc["trace_pat_4_1_8"] = buf.value.decode()
    s = np.array(ref_schedule(0, O.PAT, 8, 4), np.int32)
    R.ref_trace_csv(s.ctypes.data_as(O.I32P), len(s), 1 << 20, buf, 1 << 16)
    misc["trace_pat_8_4_1MiB"] = buf.value.decode()
    tfb = []
    mib = 1 << 20
    for b, c, n in [(4 * mib, mib, 16), (mib, mib, 16), (100 * mib, mib, 8), (mib - 1, mib, 8),
                    (3 * mib, mib, 8), (8 * mib, mib, 3), (0, 1, 2)]:
        t = ctypes.c_int()
        rc = R.ref_trees_from_buffer(b, c, n, ctypes.byref(t))
        tfb.append({"buffer": b, "chunk": c, "n": n, "rc": rc, "trees": t.value if rc == 0 else None})
    misc["trees_from_buffer"] = tfb
    rcf = []
    for n, t in [(8, 2), (16, 8), (16, 1), (12, 2), (16, 3), (256, 128), (2, 1)]:
        v = ctypes.c_int()
        rc = R.ref_round_count_formula(n, t, ctypes.byref(v))
        rcf.append({"n": n, "trees": t, "rc": rc, "rounds": v.value if rc == 0 else None})
    misc["round_count_formula"] = rcf
    mm = ctypes.c_int64()
    R.ref_oracle_sweep(1, 64, 4, ctypes.byref(mm))
    misc["reference_oracle_sweep_1_64_mismatches"] = mm.value
    with open(os.path.join(OUT, "misc.json"), "w") as f:
        json.dump(misc, f, indent=1)
    print("wrote", len(scheds), "schedules,", len(index), "executor cases")


if __name__ == "__main__":
    main()

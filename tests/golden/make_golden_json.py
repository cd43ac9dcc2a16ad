"""Golden fixtures for the schedule JSON format, from the REFERENCE ITSELF (serialize.cpp:49-101,
compiled into oracle/_ref/libpatsim_ref.so with the image's nlohmann json.hpp v3.11.3).

    make -C oracle ref && python tests/golden/make_golden_json.py

Writes tests/golden/schedule_json.json:
  "dumps":  reference schedule_to_json text (indent 2 and compact) for every generator, kind,
            n in {1..8, 12, 16} and every valid T
  "parses": documents (valid and malformed) with the reference schedule_from_json outcome:
            the flat-encoded schedule, or the ParseError message
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


def main():
    R = O.ref()
    R.ref_schedule_to_json.argtypes = [O.I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]
    R.ref_schedule_to_json.restype = ctypes.c_int64
    R.ref_schedule_from_json.argtypes = [ctypes.c_char_p, O.I32P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    dumps = []
    for n in list(range(1, 9)) + [12, 16]:
        for kind in (O.ALLGATHER, O.REDUCESCATTER):
            for algo in range(5):
                if algo == O.RECURSIVE_DOUBLING and n & (n - 1):
                    continue
                for t in (O.valid_tree_counts(n) if algo == O.PAT else [0]):
                    s = O.schedule(kind, algo, n, t)
                    for indent in (2, -1):
                        buf = ctypes.create_string_buffer(1 << 16)
                        ln = R.ref_schedule_to_json(s.ctypes.data_as(O.I32P), len(s), indent, buf, 1 << 16)
                        assert ln > 0
                        dumps.append({"schedule": [int(x) for x in s], "indent": indent, "text": buf.value.decode()})
    base = json.loads(dumps[-1]["text"])
    docs = {
        "readme_example": '{"algorithm": "pat", "kind": "allgather", "n_ranks": 8, "params": {"trees": 2, '
                          '"buffer_slots": 4}, "rounds": [{"round": 0, "dim": 2, "split": 0, "peer": 4, "chunks": [0]}]}',
        "ring_no_params": json.dumps({"algorithm": "ring", "kind": "reducescatter", "n_ranks": 3, "params": {},
                                      "rounds": [{"round": 0, "dim": 0, "split": 0, "peer": -1, "chunks": [1]}]}),
        "rd_exchange": json.dumps({"algorithm": "recursive-doubling", "kind": "allgather", "n_ranks": 4, "params": {},
                                   "rounds": [{"round": 0, "dim": 0, "split": 0, "peer": 1, "chunks": [0]}]}),
        "malformed": '{"algorithm": "pat", ',
        "missing_kind": json.dumps({"algorithm": "pat", "n_ranks": 8, "params": {}, "rounds": []}),
        "bad_algorithm": json.dumps({**base, "algorithm": "tree"}),
        "bad_kind": json.dumps({**base, "kind": "allreduce"}),
        "params_not_object": json.dumps({**base, "params": [1, 2]}),
        "params_missing_slots": json.dumps({**base, "params": {"trees": 2}}),
        "rounds_not_array": json.dumps({**base, "rounds": {}}),
        "round_missing_peer": json.dumps({**base, "rounds": [{"round": 0, "dim": 0, "split": 0, "chunks": [0]}]}),
        "wrong_type_n": json.dumps({**base, "n_ranks": "eight"}),
        "wrong_type_chunks": json.dumps({**base, "rounds": [{"round": 0, "dim": 0, "split": 0, "peer": 1, "chunks": "0"}]}),
    }
    parses = {}
    for name, text in docs.items():
        out = np.zeros(1 << 14, np.int32)
        ln = ctypes.c_int64()
        rc = R.ref_schedule_from_json(text.encode(), out.ctypes.data_as(O.I32P), len(out), ctypes.byref(ln))
        parses[name] = {"text": text, "rc": rc,
                        "error": O.ERRORS.get(rc) if rc else None,
                        "message": R.ref_last_error().decode() if rc else None,
                        "schedule": [int(x) for x in out[: ln.value]] if rc == 0 else None}
    with open(os.path.join(OUT, "schedule_json.json"), "w") as f:
        json.dump({"generator": "oracle/_ref/libpatsim_ref.so (reference serialize.cpp)", "dumps": dumps,
                   "parses": parses}, f, indent=1)
    print("wrote", len(dumps), "dumps and", len(parses), "parse cases")


if __name__ == "__main__":
    main()

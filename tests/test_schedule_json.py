"""The reference's schedule file format (serialize.cpp:49-101): our writer produces the
reference's exact text and our reader its exact results and ParseError messages, pinned to
fixtures generated from the reference itself (tests/golden/make_golden_json.py)."""
import json
import os

import pytest

from paper_2506_20252_b200 import schedule as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_json.json")))


def test_writer_matches_reference_text():
    assert len(GOLDEN["dumps"]) > 200
    for case in GOLDEN["dumps"]:
        s = S.RelativeSchedule.decode(case["schedule"])
        assert S.schedule_to_json(s, case["indent"]) == case["text"], case["schedule"][:8]


def test_reader_round_trips_every_reference_dump():
    for case in GOLDEN["dumps"]:
        assert list(S.schedule_from_json(case["text"]).encode()) == case["schedule"]


@pytest.mark.parametrize("name", sorted(GOLDEN["parses"]))
def test_reader_matches_reference_outcome(name):
    case = GOLDEN["parses"][name]
    if case["rc"] == 0:
        assert list(S.schedule_from_json(case["text"]).encode()) == case["schedule"]
    else:
        with pytest.raises(S.ParseError) as e:
            S.schedule_from_json(case["text"])
        assert str(e.value) == case["message"]


def test_imported_schedule_is_validated():
    """A schedule read from a file is checked like a generated one (schedule.cpp:194-212)."""
    pat = S.schedule_from_json(S.schedule_to_json(S.pat_allgather(8, 2)))
    assert S.validate(pat)[0] == 0
    partial = S.schedule_from_json(GOLDEN["parses"]["readme_example"]["text"])  # one round only
    assert S.validate(partial)[0] > 0

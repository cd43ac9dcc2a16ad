"""CPU property tests of the LL32 line layout (csrc/transport.cuh: LL32Shape, load_units,
store_units, ll32_phase; csrc/comm.cpp: ll32_group, shape). A restatement of the index math,
checked for every slice length a call can produce:

* the units of the non-empty lines cover the slice bytes exactly once;
* a line is empty exactly when its first unit starts past the slice end, and then every later
  line of the same lane is empty too (sender and receiver skip the same lines);
* a slice of at most the slot's payload capacity fits the slot's lines;
* a unit never straddles a slice boundary when slices are multiples of 16 bytes.
"""
import pytest

SLOT = 32 << 10


def shape(U):
    R = 7 if U == 4 else 3
    return R, 32 * R * U


def layout(L, U):
    R, G = shape(U)
    nlines = -(-L // G) * 32
    cover = [0] * L
    empty = []
    for q in range(nlines):
        gb, lane = (q >> 5) * G, q & 31
        is_empty = gb + U * lane >= L
        empty.append(is_empty)
        if is_empty:
            continue
        for r in range(R):
            off = gb + U * (32 * r + lane)
            if off < L:
                for b in range(off, min(off + U, L)):
                    cover[b] += 1
    return nlines, cover, empty


@pytest.mark.parametrize("U", [4, 8])
def test_units_cover_the_slice_exactly_once(U):
    R, G = shape(U)
    for L in list(range(0, 3 * G + 70, 4 if U == 4 else 8)) + [SLOT // 1024 * G]:
        nlines, cover, empty = layout(L, U)
        assert all(c == 1 for c in cover), (U, L)
        assert nlines * 32 <= max(SLOT, 32 * 32) or L > SLOT // 1024 * G, (U, L)
        # the first unit of a line is the lowest: a line without it has no bytes at all
        for q, e in enumerate(empty):
            if e:
                for q2 in range(q, nlines, 32):  # same lane, later groups
                    assert empty[q2], (U, L, q, q2)


@pytest.mark.parametrize("U", [4, 8])
def test_slot_capacity(U):
    _, G = shape(U)
    cap = SLOT // 1024 * G  # comm.cpp shape(): (ll32_slot_bytes / 1024) * ll32_group
    nlines, _, _ = layout(cap, U)
    assert nlines * 32 == SLOT
    nlines, _, _ = layout(cap + 4, U)
    assert nlines * 32 > SLOT  # one more byte would not fit: the host never slices past cap


def test_units_do_not_straddle_16_byte_slice_boundaries():
    # slices are multiples of 16 bytes (comm.cpp shape), units are 4 or 8 bytes at multiples of U
    for U in (4, 8):
        R, G = shape(U)
        for lane in range(32):
            for r in range(R):
                off = U * (32 * r + lane)
                assert off % U == 0 and (off % 16) + U <= 16

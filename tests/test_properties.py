"""Property-based tests (hypothesis, CPU only): the host build against the oracle
on generated FIBs, the layout walk, and the reference file-format readers under
arbitrary corruption (they must reject, never crash or mis-parse)."""
import struct

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from _util import rules_array

MASK64 = (1 << 64) - 1
SETTINGS = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def fibs(draw, max_rules=40):
    """Unique (top64, len) rules, lengths 0..64, canonical, none touching the sentinel;
    nesting comes from drawing many short tops in a small space."""
    n = draw(st.integers(0, max_rules))
    space_bits = draw(st.sampled_from([8, 16, 64]))
    seen, rules = set(), []
    for _ in range(n):
        ln = draw(st.integers(0, 64))
        top = draw(st.integers(0, (1 << space_bits) - 1)) << (64 - space_bits)
        keep = (MASK64 << (64 - ln)) & MASK64 if ln else 0
        top &= keep
        if (top, ln) in seen or top == MASK64 or top + (1 << (64 - ln)) == MASK64:
            continue
        seen.add((top, ln))
        rules.append((top << 64, ln, draw(st.integers(1, 1000))))
    return rules, draw(st.integers(0, 1000))


@pytest.fixture(scope="module")
def dtype():
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    return PREFIX_DTYPE


@SETTINGS
@given(fibs(), st.booleans())
def test_build_intervals_matches_oracle(lpm, orc, dtype, fib_def, merge):
    rules, dflt = fib_def
    arr = rules_array(rules, dtype)
    fib = lpm.FibTable(dflt, arr)
    imap = lpm.build_intervals(fib, merge_adjacent=merge)
    st_, b, nh = orc.build_intervals(arr, dflt, merge)
    assert st_ == 0
    np.testing.assert_array_equal(imap.boundaries, b)
    np.testing.assert_array_equal(imap.next_hops, nh)
    assert len(imap) <= 2 * len(rules) + 1 and imap.boundaries[0] == 0
    assert np.all(imap.boundaries[1:] > imap.boundaries[:-1])


@SETTINGS
@given(fibs(max_rules=200), st.lists(st.integers(0, MASK64), min_size=1, max_size=64))
def test_layout_walk_matches_oracle(lpm, orc, dtype, fib_def, keys):
    """The B200 layout walked exactly as the kernel walks it (test_host.walk_layout)."""
    from test_host import walk_layout
    from _util import addrs_from_keys, boundary_probe_keys
    rules, dflt = fib_def
    fib = lpm.FibTable(dflt, rules_array(rules, dtype))
    imap = lpm.build_intervals(fib)
    tree = lpm.build_tree(imap)
    k = np.concatenate([np.array(keys, np.uint64), boundary_probe_keys(imap.boundaries)])
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(k), threads=1)
    np.testing.assert_array_equal(walk_layout(tree, k), want)


@settings(max_examples=150, deadline=None)
@given(st.data())
def test_snapshot_reader_rejects_corruption(lpm, data):
    """Random byte edits / truncations of a valid PBT1 image: the reader either
    returns an interval map that re-encodes to the same bytes, or raises
    BadSnapshotFile — never anything else."""
    b = np.arange(0, 3000, 7, dtype=np.uint64) * 1000
    nh = (np.arange(len(b)) % 5 + 1).astype(np.uint32)
    img = bytearray(lpm.encode_snapshot(lpm.IntervalMap(b, nh, 0), 8))
    n_edits = data.draw(st.integers(1, 4))
    for _ in range(n_edits):
        pos = data.draw(st.integers(0, len(img) - 1))
        img[pos] = data.draw(st.integers(0, 255))
    if data.draw(st.booleans()):
        img = img[: data.draw(st.integers(0, len(img)))]
    try:
        imap, k = lpm.decode_snapshot(bytes(img))
    except lpm.Lpm6Error as e:
        assert e.code == "BadSnapshotFile", e
        return
    assert lpm.encode_snapshot(imap, k) == bytes(img)


@settings(max_examples=150, deadline=None)
@given(st.binary(max_size=64))
def test_trace_reader_rejects_garbage(lpm, blob):
    data = b"PBTR" + blob if blob[:1] != b"!" else blob
    try:
        n = lpm.trace_count(data)
    except lpm.Lpm6Error as e:
        assert e.code == "BadTraceFile"
        return
    assert len(data) == 16 + 8 * n and struct.unpack_from("<H", data, 4)[0] == 1


@settings(max_examples=200, deadline=None)
@given(st.text(max_size=60))
def test_update_parser_never_crashes(lpm, line):
    from paper_2604_14650_b200 import store
    try:
        op = store.parse_update(line)
    except lpm.Lpm6Error as e:
        assert e.code in ("MalformedAddress", "UnsupportedPrefixLength", "MissingNextHop", "ReservedNextHop")
        return
    assert op.kind in (store.ANNOUNCE, store.DELETE) and 0 <= op.prefix.length <= 64

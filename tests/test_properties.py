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


# ---- rule text: our parser against libc inet_pton (the reference's parser, fib.cpp:47) ----

_HEX = "0123456789abcdefABCDEF"


@st.composite
def address_texts(draw):
    """Valid RFC 4291 forms (full, '::'-compressed, embedded dotted quads) and near-misses."""
    groups = [draw(st.integers(0, 0xFFFF)) for _ in range(8)]
    style = draw(st.integers(0, 5))
    g = [format(x, "x") if draw(st.booleans()) else format(x, "04X") for x in groups]
    if style == 0:
        return ":".join(g)
    if style == 1:  # compress a run
        a = draw(st.integers(0, 8))
        b = draw(st.integers(a, 8))
        return ":".join(g[:a]) + "::" + ":".join(g[b:])
    if style == 2:  # dotted-quad tail
        quad = ".".join(str(draw(st.integers(0, 255))) for _ in range(4))
        if draw(st.booleans()):
            return ":".join(g[:6]) + ":" + quad
        a = draw(st.integers(0, 6))
        return ":".join(g[:a]) + "::" + quad
    # near-misses: random short strings over the address alphabet
    return draw(st.text(alphabet=_HEX + ":.x/ ", min_size=0, max_size=20))


@SETTINGS
@given(text=address_texts(), length=st.integers(0, 130), hop=st.integers(0, (1 << 32) + 5))
def test_parse_prefix_matches_inet_pton(lpm, text, length, hop):
    """lpm6_parse_prefix accepts exactly the addresses libc's inet_pton accepts (the
    reference parses with inet_pton, fib.cpp:47) and yields the same 128-bit value."""
    import socket
    try:
        raw = socket.inet_pton(socket.AF_INET6, text)
    except (OSError, ValueError):
        raw = None
    rule = f"{text}/{length} {hop}"
    if raw is None or " " in text or "/" in text or text == "":
        if raw is None:
            with pytest.raises(lpm.Lpm6Error):
                lpm.parse_prefix(rule)
        return
    value = int.from_bytes(raw, "big")
    if length > 128:
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.parse_prefix(rule)
        assert e.value.code == "MalformedAddress"
        return
    if length > 64:
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.parse_prefix(rule)
        assert e.value.code == "UnsupportedPrefixLength"
        return
    if hop > 0xFFFFFFFF:
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.parse_prefix(rule)
        assert e.value.code == "MissingNextHop"
        return
    if hop == 0xFFFFFFFF:
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.parse_prefix(rule)
        assert e.value.code == "ReservedNextHop"
        return
    p, masked = lpm.parse_prefix(rule)
    keep = ((1 << 128) - 1) ^ ((1 << (128 - length)) - 1)
    assert p.value == value & keep and p.length == length and p.next_hop == hop
    assert masked == ((value & keep) != value)


@pytest.mark.parametrize("text", ["2001:db8::/32 1", "::/0 7", "::ffff:10.0.0.1/64 9", "1:2:3:4:5:6:7::/48 2",
                                  "::1:2:3:4:5:6:7/64 3", "2001:DB8:0:0:1::/64 5"])
def test_parse_prefix_matches_reference(lpm, ref, text):
    """Against the reference's own parse_prefix (oracle/_ref, fib.cpp:72-105)."""
    import ctypes
    buf = np.zeros(1, lpm.fib.PREFIX_DTYPE)
    masked = ctypes.c_int(0)
    st_ = ref.L.ref_parse_prefix(text.encode(), buf.ctypes.data, ctypes.byref(masked))
    assert st_ == 0
    p, m = lpm.parse_prefix(text)
    assert p.value == (int(buf["value_hi"][0]) << 64 | int(buf["value_lo"][0]))
    assert p.length == int(buf["length"][0]) and p.next_hop == int(buf["next_hop"][0]) and m == bool(masked.value)

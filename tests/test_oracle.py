"""Pin the CPU oracle (oracle/lpm6_oracle.c) and the product's host build.

* SPEC known-answer vectors — transcribed from the spec's examples.
* Golden fixtures produced by the reference itself (tests/golden/make_golden.py,
  oracle/_ref: the reference's fib.cpp + intervals.cpp).
* Oracle properties: interval oracle == linear oracle, variant
  equivalence of the restated searches, interval bounds.
"""
from pathlib import Path

import numpy as np
import pytest

from _util import MASK64, addrs_from_keys, boundary_probe_keys, large_rules, random_fib_rules, rules_array, sha

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith("large_"))
LARGE_FIXTURES = sorted(p.stem for p in GOLDEN.glob("large_*.npz"))

A = 0x20010DB800000000        # 2001:db8::
B = 0x20010DB800010000        # 2001:db8:1::
BEND = 0x20010DB800020000
AEND = 0x20010DB900000000
S = MASK64


@pytest.fixture(scope="module")
def spec_rules():
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    return rules_array([(A << 64, 32, 1), (B << 64, 48, 2)], PREFIX_DTYPE)


# ---- SPEC known-answer tests ------------------------------------------------------------------

def test_parse_prefix_kat(lpm):
    p, masked = lpm.parse_prefix("2001:db8::/32 1")
    assert (p.value, p.length, p.next_hop, masked) == (A << 64, 32, 1, False)
    p, _ = lpm.parse_prefix("::/0 7")
    assert (p.value, p.length, p.next_hop) == (0, 0, 7)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.parse_prefix("2001:db8::/96 3")
    assert e.value.code == "UnsupportedPrefixLength"
    p, masked = lpm.parse_prefix("2001:db8::1/32 4")                       # host bits masked
    assert p.value == A << 64 and masked
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.parse_prefix("2001:db8::/32")
    assert e.value.code == "MissingNextHop"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.parse_prefix("2001:zz8::/32 1")
    assert e.value.code == "MalformedAddress"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.parse_prefix("::/0 4294967295")
    assert e.value.code == "ReservedNextHop"


def test_prefix_to_range_kat(ref):
    import ctypes as C
    from oracle.oracle import U64
    from paper_2604_14650_b200.fib import PREFIX_DTYPE

    def rng_of(v, ln):
        r = rules_array([(v, ln, 1)], PREFIX_DTYPE)
        s, eh, el = U64(), U64(), U64()
        ref.L.ref_prefix_to_range(r.ctypes.data, C.byref(s), C.byref(eh), C.byref(el))
        return s.value, (eh.value << 64) | el.value

    assert rng_of(A << 64, 32) == (A, AEND)
    assert rng_of(0, 0) == (0, 1 << 64)
    assert rng_of(B << 64, 48) == (B, BEND)


def test_build_intervals_kat(lpm, orc, spec_rules):
    want_b = np.array([0, A, B, BEND, AEND], np.uint64)
    want_nh = np.array([0, 1, 2, 1, 0], np.uint32)
    st, b, nh = orc.build_intervals(spec_rules, 0)
    assert st == 0
    np.testing.assert_array_equal(b, want_b)
    np.testing.assert_array_equal(nh, want_nh)
    im = lpm.build_intervals(lpm.FibTable(0, spec_rules))
    np.testing.assert_array_equal(im.boundaries, want_b)
    np.testing.assert_array_equal(im.next_hops, want_nh)
    assert len(b) == 2 * 2 + 1
    st, b, nh = orc.build_intervals(spec_rules[:0], 3)
    assert list(b) == [0] and list(nh) == [3]
    assert list(lpm.build_intervals(lpm.FibTable(3)).boundaries) == [0]


def test_linear_and_interval_oracle_kat(orc, spec_rules):
    assert orc.lookup_linear(spec_rules, 0, (A << 64) | (1 << 48)) == 1            # S:139 (2001:db8:0:0:1::)
    assert orc.lookup_linear(spec_rules, 0, (B << 64) | 5) == 2
    assert orc.lookup_linear(spec_rules[:0], 77, 0x9999 << 112) == 77
    st, b, nh = orc.build_intervals(spec_rules, 0)
    assert orc.lookup_interval(b, nh, 0x20010DB800015000) == 2
    assert orc.lookup_interval(b, nh, 0) == 0
    assert orc.lookup_interval(b, nh, MASK64 - 1) == nh[-1]


def test_geometry_kat(orc):
    g = orc.plan_geometry(472392, 8)
    assert g.depth == 5 and g.b ** 5 == 59049
    g = orc.plan_geometry(5, 8)
    assert g.depth == 0 and g.leaf_start == 0
    g = orc.plan_geometry(100, 8)
    assert g.depth == 2 and list(g.level_start[:3]) == [0, 8, 80] and g.allocated_leaf_nodes == 13
    g1 = orc.plan_geometry(1000, 8)
    assert orc.child_key_start(g1, 0, 0, 0) == 8
    assert orc.child_key_start(g1, 0, 0, 2) == 24
    assert orc.child_key_start(g1, 1, 3, 0) == 80 + 27 * 8


def test_build_tree_kat(orc, spec_rules):
    st, b, nh = orc.build_intervals(spec_rules, 0)
    g, keys, values = orc.build_tree(b, nh, 8)
    assert g.depth == 0
    assert list(keys[:8]) == [0, A, B, BEND, AEND, S, S, S]
    assert list(values) == [0, 1, 2, 1, 0, 0, 0, 0]
    b100 = np.arange(100, dtype=np.uint64) * 1000
    g, keys, values = orc.build_tree(b100, np.arange(100, dtype=np.uint32), 8)
    assert orc.L.orc_total_key_slots(__import__("ctypes").byref(g)) == 80 + 13 * 8
    assert list(keys[8:16]) == [b100[8 * (j + 1)] for j in range(8)]     # level 1 node 0 separators
    # S:230 / S:488: full depth-5 k=8 tree: leaf 8*9^5*8 bytes, internal 8*level_start(5)
    g = orc.plan_geometry(472392, 8)
    assert 8 * 9 ** 5 * 8 == 3779136 and 8 * g.level_start[5] == 472384


def test_search_kat(orc, spec_rules):
    st, b, nh = orc.build_intervals(spec_rules, 0)
    g, keys, values = orc.build_tree(b, nh, 8)
    assert orc.search_scalar(keys, g, 0x20010DB800015000) == 2            # S:283 (rank 3 - 1)
    assert orc.search_scalar(keys, g, 0) == 0
    assert orc.search_branchfree(keys, g, MASK64) == len(b) - 1           # S:316 clamp
    b100 = np.arange(100, dtype=np.uint64) * 1000 + 7
    b100[0] = 0
    g, keys, values = orc.build_tree(b100, np.arange(100, dtype=np.uint32), 8)
    assert orc.search_scalar(keys, g, int(b100[57])) == 57
    for i in range(100):
        for k in (int(b100[i]), int(b100[i]) + 1, max(int(b100[i]) - 1, 0)):
            assert orc.search_branchfree(keys, g, k) == orc.search_scalar(keys, g, k)


# ---- golden fixtures from the reference ---------------------------------------------------------

@pytest.mark.parametrize("name", FIXTURES)
def test_golden_oracle(orc, lpm, name):
    d = np.load(GOLDEN / f"{name}.npz")
    rules, dflt = d["rules"], int(d["default_nh"][0])
    for merge in (1, 0):
        st, b, nh = orc.build_intervals(rules, dflt, bool(merge))
        assert st == 0
        np.testing.assert_array_equal(b, d[f"boundaries_m{merge}"])
        np.testing.assert_array_equal(nh, d[f"next_hops_m{merge}"])
        im = lpm.build_intervals(lpm.FibTable(dflt, rules), merge_adjacent=bool(merge))
        np.testing.assert_array_equal(im.boundaries, d[f"boundaries_m{merge}"])
        np.testing.assert_array_equal(im.next_hops, d[f"next_hops_m{merge}"])
    st, b, nh = orc.build_intervals(rules, dflt, True)
    out, _ = orc.lookup_batch(0, b, nh, addrs_from_keys(d["keys"]), threads=4)
    np.testing.assert_array_equal(out, d["interval_oracle"])
    if "linear_oracle" in d:
        np.testing.assert_array_equal(out, d["linear_oracle"])
    for variant in (1, 2):
        got, _ = orc.lookup_batch(variant, b, nh, addrs_from_keys(d["keys"]), threads=2)
        np.testing.assert_array_equal(got, d["interval_oracle"])


@pytest.mark.parametrize("name", LARGE_FIXTURES)
def test_golden_large_oracle(orc, lpm, name):
    """Hash-pinned reference fixtures at SPEC acceptance size (10^5 rules) and
    the deepest tree (the 1M-prefix C2 FIB): the rules are regenerated from their
    recorded source and must match their sha256; the restatement's and the product's
    interval maps must hash to the reference's (merge on and off); sampled keys must
    get the reference's interval-oracle and linear-oracle answers."""
    d = np.load(GOLDEN / f"{name}.npz")
    rules, dflt = large_rules(d)
    for merge in (1, 0):
        st, b, nh = orc.build_intervals(rules, dflt, bool(merge))
        assert st == 0 and len(b) == int(d[f"m_m{merge}"][0])
        assert sha(b) == str(d[f"boundaries_sha256_m{merge}"]) and sha(nh) == str(d[f"next_hops_sha256_m{merge}"])
        im = lpm.build_intervals(lpm.FibTable(dflt, rules), merge_adjacent=bool(merge))
        assert sha(im.boundaries) == str(d[f"boundaries_sha256_m{merge}"])
        assert sha(im.next_hops) == str(d[f"next_hops_sha256_m{merge}"])
    st, b, nh = orc.build_intervals(rules, dflt, True)
    out, _ = orc.lookup_batch(0, b, nh, addrs_from_keys(d["keys"]), threads=8)
    np.testing.assert_array_equal(out, d["interval_oracle"])
    pos = np.searchsorted(d["keys"], d["linear_keys"])
    np.testing.assert_array_equal(out[pos], d["linear_oracle"])


def test_reference_agrees_with_restatement(ref, orc, lpm):
    """Live check against the compiled reference on the workload FIBs (C0, C1 and the
    1M-prefix C2 FIB)."""
    for kind in (0, 1, 2):
        fib = lpm.workload_fib(kind)
        st, m = ref.build_intervals(fib.rules, fib.default_next_hop)
        assert st == 0
        st, b, nh = orc.build_intervals(fib.rules, fib.default_next_hop)
        np.testing.assert_array_equal(b, m.boundaries)
        np.testing.assert_array_equal(nh, m.next_hops)
        keys = boundary_probe_keys(b)[:200000]
        out, _ = orc.lookup_batch(0, b, nh, addrs_from_keys(keys), threads=8)
        np.testing.assert_array_equal(out, m.lookup(keys, 8))


# ---- oracle properties ------------------------------------------------------------------------

def test_interval_equals_linear_oracle(orc):
    """interval oracle == brute-force LPM on random and boundary+-1 addresses."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(7)
    for n, dflt in ((50, True), (400, False)):
        rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.5)
        st, b, nh = orc.build_intervals(rules, 11)
        keys = np.concatenate([boundary_probe_keys(b), rng.integers(0, 2**64, 3000, dtype=np.uint64)])
        addrs = addrs_from_keys(keys, rng)
        got, _ = orc.lookup_batch(0, b, nh, addrs, threads=4)
        for i in range(0, len(addrs), 7):
            a = (int(addrs[i, 1]) << 64) | int(addrs[i, 0])
            assert got[i] == orc.lookup_linear(rules, 11, a)


def test_variant_equivalence_restated_search(orc, lpm):
    """scalar / branch-free / AVX-512 batched restatements agree on >= 1e5 keys."""
    fib = lpm.workload_fib(1)
    st, b, nh = orc.build_intervals(fib.rules, fib.default_next_hop)
    rng = np.random.default_rng(3)
    keys = np.concatenate([boundary_probe_keys(b)[:60000], rng.integers(0, 2**64, 60000, dtype=np.uint64)])
    addrs = addrs_from_keys(keys)
    tree = orc.build_tree(b, nh, 8)
    want, _ = orc.lookup_batch(0, b, nh, addrs, threads=8)
    for variant in (1, 2):
        got, ran = orc.lookup_batch(variant, b, nh, addrs, threads=8, tree=tree)
        np.testing.assert_array_equal(got, want)


def test_interval_count_bounds(lpm):
    """for 1,000 random FIBs (N <= 1000): m <= 2N+1, strictly increasing, starts at 0."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(11)
    for i in range(1000):
        n = int(rng.integers(0, 60)) if i < 900 else int(rng.integers(0, 1001))
        rules = random_fib_rules(rng, n, PREFIX_DTYPE, bool(i & 1), nest_p=0.4)
        for merge in (True, False):
            im = lpm.build_intervals(lpm.FibTable(3, rules), merge_adjacent=merge)
            assert len(im) <= 2 * len(rules) + 1
            assert im.boundaries[0] == 0
            assert np.all(np.diff(im.boundaries.astype(np.float64)) >= 0)
            assert np.all(im.boundaries[1:] > im.boundaries[:-1])
            assert not np.any(im.boundaries == np.uint64(MASK64))


def test_build_errors(lpm, orc):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    # ReservedNextHop (intervals.cpp:36-37)
    r = rules_array([(A << 64, 32, 0xFFFFFFFF)], PREFIX_DTYPE)
    assert orc.build_intervals(r, 0)[0] == 4
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.build_intervals(lpm.FibTable(0, r))
    assert e.value.code == "ReservedNextHop"
    # SentinelCollision (intervals.cpp:76-79): a /64 starting at or ending on ffff:ffff:ffff:ffff
    for top in (MASK64, MASK64 - 1):
        r = rules_array([(top << 64, 64, 3)], PREFIX_DTYPE)
        assert orc.build_intervals(r, 0)[0] == 7
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.build_intervals(lpm.FibTable(0, r))
        assert e.value.code == "SentinelCollision"
    # a collision is an error even when merging would drop that boundary (checked before merge)
    r = rules_array([(0, 0, 3), ((MASK64 - 1) << 64, 64, 3)], PREFIX_DTYPE)
    assert orc.build_intervals(r, 0)[0] == 7
    with pytest.raises(lpm.Lpm6Error):
        lpm.build_intervals(lpm.FibTable(0, r))
    # DuplicatePrefix, UnsupportedPrefixLength, non-canonical (product rejects)
    r = rules_array([(A << 64, 32, 1), (A << 64, 32, 2)], PREFIX_DTYPE)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.build_intervals(lpm.FibTable(0, r))
    assert e.value.code == "DuplicatePrefix"
    r = rules_array([(A << 64, 65, 1)], PREFIX_DTYPE)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.build_intervals(lpm.FibTable(0, r))
    assert e.value.code == "UnsupportedPrefixLength"
    r = rules_array([((A | 1) << 64, 32, 1)], PREFIX_DTYPE)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.build_intervals(lpm.FibTable(0, r))
    assert e.value.code == "InvalidArgument"


def test_merge_on_off_same_answers(orc):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(5)
    rules = random_fib_rules(rng, 500, PREFIX_DTYPE, True, nest_p=0.6)
    rules["next_hop"] = rng.integers(1, 4, len(rules))  # few next hops -> many merges
    st1, b1, nh1 = orc.build_intervals(rules, 2, True)
    st0, b0, nh0 = orc.build_intervals(rules, 2, False)
    assert len(b1) < len(b0)
    keys = np.concatenate([boundary_probe_keys(b0), rng.integers(0, 2**64, 5000, dtype=np.uint64)])
    a, _ = orc.lookup_batch(0, b1, nh1, addrs_from_keys(keys))
    c, _ = orc.lookup_batch(0, b0, nh0, addrs_from_keys(keys))
    np.testing.assert_array_equal(a, c)

"""Update engine on the host (no GPU): trace parsing and the store's staging rule
(csrc/lpm6/update.cpp via lpm6_parse_update / lpm6_apply_updates) against the
pure-Python restatement oracle/update_oracle.py and the SPEC's examples."""
import numpy as np
import pytest

from oracle import update_oracle as U
from _util import random_fib_rules

MASK64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def st():
    from paper_2604_14650_b200 import store
    return store


def op(st, kind, v, ln, nh=0):
    from paper_2604_14650_b200.fib import Prefix
    return st.UpdateOp(kind, Prefix(v, ln, nh))


def rule_set(fib):
    return sorted((int(r["value_hi"]) << 64 | int(r["value_lo"]), int(r["length"]), int(r["next_hop"]))
                  for r in fib.rules)


# ---- trace format -------------------------------------------------------------------------

def test_parse_update_lines(st):
    a = st.parse_update("A 2001:db8::/32 7")
    assert (a.kind, a.prefix.length, a.prefix.next_hop) == (st.ANNOUNCE, 32, 7)
    assert a.prefix.value == 0x20010DB8 << 96
    w = st.parse_update("W 2001:db8:1::/48")
    assert (w.kind, w.prefix.length, w.prefix.next_hop) == (st.DELETE, 48, 0)
    w2 = st.parse_update("  W 2001:db8:1::/48 9  ")  # next hop allowed and ignored on withdraw
    assert w2 == w
    m = st.parse_update("A 2001:db8::1/32 5")  # host bits masked as parse_prefix does
    assert m.prefix.value == 0x20010DB8 << 96


@pytest.mark.parametrize("line,code", [
    ("X 2001:db8::/32 7", "MalformedAddress"),
    ("A2001:db8::/32 7", "MalformedAddress"),
    ("A 2001:db8::/80 7", "UnsupportedPrefixLength"),
    ("A 2001:db8::/32", "MissingNextHop"),
    ("A 2001:db8::/32 4294967295", "ReservedNextHop"),
    ("A 2001:zz8::/32 1", "MalformedAddress"),
])
def test_parse_update_errors(st, line, code):
    from paper_2604_14650_b200 import Lpm6Error
    with pytest.raises(Lpm6Error) as e:
        st.parse_update(line)
    assert e.value.code == code


def test_parse_update_matches_oracle(st):
    rng = np.random.default_rng(3)
    for _ in range(300):
        ln = int(rng.integers(0, 65))
        v = int(rng.integers(0, 2**63)) << 65 | int(rng.integers(0, 2**63))
        import ipaddress
        text = str(ipaddress.IPv6Address(v))
        line = f"A {text}/{ln} {int(rng.integers(0, 1000))}" if rng.random() < 0.5 else f"W {text}/{ln}"
        want = U.parse_update_line(line)
        got = st.parse_update(line)
        assert (got.kind, got.prefix.value, got.prefix.length, got.prefix.next_hop) == want


def test_load_update_trace_counts_bad_lines(st):
    text = "# header\nA 2001:db8::/32 1\n\nW 2001:db8::/32\nbogus line\nA ::/0 3  # default\nA 1::/90 1\n"
    ops, errors = st.load_update_trace(text)
    assert len(ops) == 3 and errors == 2
    assert [o.kind for o in ops] == [st.ANNOUNCE, st.DELETE, st.ANNOUNCE]


# ---- staging rule ----------------------------------------------------------------------

def test_spec_stage_examples(lpm, st):
    base = lpm.FibTable(0)
    p = 0x20010DB8 << 96
    # stage 100 inserts -> staged = 100
    ins = [op(st, st.INSERT, (0x2001 << 112) | (i << 64), 64, i + 1) for i in range(100)]
    fib, staged, errs = st.apply_updates(base, ins)
    assert staged == 100 and errs == [None] * 100 and len(fib) == 100
    # delete of an absent prefix -> staged = 0, 1 error
    fib2, staged, errs = st.apply_updates(fib, [op(st, st.DELETE, p, 32)])
    assert staged == 0 and errs == ["UnknownPrefix"] and rule_set(fib2) == rule_set(fib)
    # insert + delete of the same prefix in one batch -> both staged, net no-op
    fib3, staged, errs = st.apply_updates(fib, [op(st, st.INSERT, p, 32, 5), op(st, st.DELETE, p, 32)])
    assert staged == 2 and errs == [None, None] and rule_set(fib3) == rule_set(fib)
    # only withdrawals of absent prefixes -> errors counted, FIB unchanged
    fib4, staged, errs = st.apply_updates(fib, [op(st, st.DELETE, p | (i << 64), 64) for i in range(5)])
    assert staged == 0 and errs.count("UnknownPrefix") == 5 and rule_set(fib4) == rule_set(fib)


def test_stage_error_codes(lpm, st):
    p = 0x20010DB8 << 96
    base, _, _ = st.apply_updates(lpm.FibTable(0), [op(st, st.INSERT, p, 32, 5)])
    cases = [
        (op(st, st.INSERT, p, 32, 6), "DuplicatePrefix"),
        (op(st, st.INSERT, p | (1 << 64), 64, 0xFFFFFFFF), "ReservedNextHop"),
        (op(st, st.MODIFY, p, 48, 6), "UnknownPrefix"),
        (op(st, st.MODIFY, p, 32, 0xFFFFFFFF), "ReservedNextHop"),
        (op(st, st.MODIFY, p, 48, 0xFFFFFFFF), "ReservedNextHop"),  # reserved checked first (fib.cpp:154)
        (op(st, st.ANNOUNCE, p, 32, 0xFFFFFFFF), "ReservedNextHop"),
        (op(st, st.INSERT, p | 1, 32, 1), "InvalidArgument"),  # host bits set
        (op(st, st.INSERT, p, 65, 1), "UnsupportedPrefixLength"),
    ]
    for o, code in cases:
        fib, staged, errs = st.apply_updates(base, [o])
        assert (staged, errs) == (0, [code]), (o, errs)
        assert rule_set(fib) == rule_set(base)
    a = np.zeros(1, st.UPDATE_DTYPE)
    a["kind"] = 9
    assert st.apply_updates(base, a)[2] == ["InvalidArgument"]
    # modify / announce change the next hop in place
    fib, staged, _ = st.apply_updates(base, [op(st, st.MODIFY, p, 32, 9)])
    assert rule_set(fib) == [(p, 32, 9)]
    fib, staged, _ = st.apply_updates(base, [op(st, st.ANNOUNCE, p, 32, 11), op(st, st.ANNOUNCE, p, 48, 12)])
    assert rule_set(fib) == [(p, 32, 11), (p, 48, 12)]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_stage_matches_oracle_on_random_streams(lpm, st, seed):
    """Random op streams (valid and invalid) over a random FIB: the C++ staging rule
    gives the oracle's rule list (same order) and per-op errors."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(seed)
    rules = random_fib_rules(rng, 400, PREFIX_DTYPE, True, nest_p=0.4)
    base = lpm.FibTable(0, rules)
    existing = [(int(r["value_hi"]) << 64, int(r["length"])) for r in rules]
    ops = []
    for _ in range(2000):
        kind = int(rng.integers(0, 4))
        if rng.random() < 0.6 and existing:
            v, ln = existing[int(rng.integers(0, len(existing)))]
        else:
            ln = int(rng.integers(0, 65))
            v = (int(rng.integers(0, 2**63)) << 1) << 64
            v &= 0 if ln == 0 else ((1 << 128) - 1) << (128 - ln) & ((1 << 128) - 1)
            existing.append((v, ln))
        nh = int(rng.integers(1, 2**20)) if rng.random() > 0.01 else 0xFFFFFFFF
        ops.append((kind, v, ln, nh))
    ofib = U.OracleFib((int(r["value_hi"]) << 64, int(r["length"]), int(r["next_hop"])) for r in rules)
    want_staged, want_errs = U.stage(ofib, ops)
    fib, staged, errs = st.apply_updates(base, [op(st, k, v, ln, nh) for k, v, ln, nh in ops])
    assert errs == want_errs
    assert staged == want_staged
    got = [(int(r["value_hi"]) << 64 | int(r["value_lo"]), int(r["length"]), int(r["next_hop"])) for r in fib.rules]
    assert got == ofib.entries


def test_store_symbols_exported(lpm):
    from paper_2604_14650_b200._lib import lib
    for name in ("lpm6cu_store_create", "lpm6cu_store_stage", "lpm6cu_store_commit", "lpm6cu_store_acquire",
                 "lpm6cu_store_release", "lpm6cu_store_destroy", "lpm6_apply_updates", "lpm6_parse_update"):
        assert hasattr(lib(), name)


def test_store_without_gpu_fails_loudly(lpm, st):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lpm.Lpm6Error) as e:
        st.FibStore(lpm.workload_fib(0))
    assert e.value.code == "CudaError"

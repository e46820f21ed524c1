"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def rules_array(prefixes, dtype):
    """[(value128, length, next_hop), ...] -> structured array in lpm6::Prefix layout."""
    a = np.zeros(len(prefixes), dtype)
    for i, (v, ln, nh) in enumerate(prefixes):
        a[i]["value_lo"] = v & MASK64
        a[i]["value_hi"] = v >> 64
        a[i]["length"] = ln
        a[i]["next_hop"] = nh
    return a


def addrs_from_keys(keys, rng=None) -> np.ndarray:
    """uint64[n,2] addresses (lo, hi) with the given top-64 keys and random low words."""
    keys = np.asarray(keys, np.uint64)
    out = np.empty((len(keys), 2), np.uint64)
    out[:, 1] = keys
    out[:, 0] = 0 if rng is None else rng.integers(0, 2**64, len(keys), dtype=np.uint64)
    return out


def boundary_probe_keys(boundaries: np.ndarray) -> np.ndarray:
    """Every boundary, boundary-1, boundary+1 plus 0 and the all-ones key."""
    b = boundaries.astype(np.uint64)
    with np.errstate(over="ignore"):
        k = np.concatenate([b, b - np.uint64(1), b + np.uint64(1),
                            np.array([0, 2**64 - 1, 2**64 - 2], np.uint64)])
    return k


def random_fib_rules(rng, n, dtype, with_default: bool, nest_p: float = 0.3, min_len: int = 0):
    """Random canonical rules, some nested, none touching the sentinel key; unique (top, len)."""
    seen = set()
    rules = []
    if with_default:
        rules.append((0, 0, int(rng.integers(1, 2**16))))
        seen.add((0, 0))
    tops = []
    while len(rules) < n + (1 if with_default else 0):
        if tops and rng.random() < nest_p:
            ptop, plen = tops[int(rng.integers(0, len(tops)))]
            if plen >= 64:
                continue
            ln = int(rng.integers(plen + 1, 65))
            extra = int(rng.integers(0, 2**63)) << 1 | int(rng.integers(0, 2))
            keep = (MASK64 << (64 - plen)) & MASK64 if plen else 0
            top = (ptop & keep) | (extra & ~keep & MASK64)
        else:
            ln = int(rng.integers(max(min_len, 1), 65))
            top = int(rng.integers(0, 2**63)) << 1 | int(rng.integers(0, 2))
        keep = (MASK64 << (64 - ln)) & MASK64 if ln else 0
        top &= keep
        end = top + (1 << (64 - ln))
        if top == MASK64 or end == MASK64 or (top, ln) in seen:
            continue
        seen.add((top, ln))
        tops.append((top, ln))
        rules.append((top << 64, ln, int(rng.integers(1, 2**16))))
    return rules_array(rules, dtype)


def sha(a: np.ndarray) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def large_fixture_rules(source: str):
    """Regenerate the rules of a hash-pinned golden fixture (make_golden.make_large)
    from its recorded source string -> (rules, default next hop)."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    kind, _, arg = source.partition(":")
    if kind == "random_nested":  # random_fib_rules(default_rng(seed), n, ..., with_default=True, nest_p=0.5)
        n, seed = (int(x) for x in arg.split(","))
        return random_fib_rules(np.random.default_rng(seed), n, PREFIX_DTYPE, True, nest_p=0.5), 7
    if kind == "ref_synth":  # the reference's synth_fib(n, seed) (fib.cpp:237-273)
        import pytest
        from oracle.oracle import REF_SO, RefOracle
        if not REF_SO.exists():
            pytest.skip("oracle/_ref not built: the reference's synth_fib regenerates this fixture")
        n, seed = (int(x) for x in arg.split(","))
        return RefOracle().synth_fib(n, seed, PREFIX_DTYPE), 0
    if kind == "workload":  # our seeded workload FIB (csrc/lpm6/workload.cpp)
        from oracle.workload import Workloads
        f = Workloads().fib(int(arg))
        return f.rules, f.default_next_hop
    raise ValueError(source)


def large_rules(d):
    """Rules of a loaded large fixture, checked against the recorded sha256."""
    rules, dflt = large_fixture_rules(str(d["source"]))
    assert len(rules) == int(d["n_rules"][0]) and sha(rules) == str(d["rules_sha256"]), "fixture rules changed"
    return rules, dflt

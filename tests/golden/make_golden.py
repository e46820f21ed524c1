"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only where the reference sources are available (this container): it uses
oracle/_ref/liblpm6ref.so — the reference's own fib.cpp + intervals.cpp compiled
in place by oracle/Makefile — to produce, for a set of FIBs:
  * the reference synth_fib rules (fib.cpp:237-273) or our random nested rules,
  * build_intervals output with merge on and off (intervals.cpp:33-93),
  * next hops of sampled keys from lookup_interval_oracle (intervals.cpp:142-145)
    and from linear_oracle_keys (intervals.cpp:109-140).
The fixtures are committed; tests/test_oracle.py pins the C restatement and the
product's host build to them without needing the reference at test time.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE.parent))

from _util import MASK64, large_fixture_rules, random_fib_rules, sha  # noqa: E402
from oracle.oracle import RefOracle  # noqa: E402
from paper_2604_14650_b200.fib import PREFIX_DTYPE  # noqa: E402


def sample_keys(rng, boundaries, n_random):
    b = boundaries.astype(np.uint64)
    with np.errstate(over="ignore"):
        k = np.concatenate([b, b - np.uint64(1), b + np.uint64(1),
                            rng.integers(0, 2**64, n_random, dtype=np.uint64),
                            np.array([0, MASK64, MASK64 - 1], np.uint64)])
    return np.unique(k)


def make(ref, name, rules, default_nh, rng, n_random=2000, linear=True):
    out = {"rules": rules, "default_nh": np.array([default_nh], np.uint32)}
    for merge in (1, 0):
        st, m = ref.build_intervals(rules, default_nh, bool(merge))
        assert st == 0, ref.error()
        out[f"boundaries_m{merge}"] = m.boundaries
        out[f"next_hops_m{merge}"] = m.next_hops
        if merge:
            keys = sample_keys(rng, m.boundaries, n_random)
            out["keys"] = keys
            out["interval_oracle"] = m.lookup(keys)
            if linear:
                out["linear_oracle"] = ref.linear_keys(rules, default_nh, keys)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, len(rules), "rules ->", len(out["boundaries_m1"]), "intervals,", len(out["keys"]), "keys")


def make_large(ref, name, rules, default_nh, rng, source, n_interval=60000, n_linear=20000):
    """Fixtures for FIBs too large to commit: the rules are regenerated at test time
    from `source` (and checked against their sha256); the reference's interval map is
    pinned by its size and sha256 (merge on and off), and its answers by sampled keys:
    boundaries / boundary+-1 / random keys through lookup_interval_oracle, and a
    subset through the brute-force linear oracle (SPEC S:486 asks 10^5 rules against
    the linear oracle)."""
    out = {"source": np.array(source), "rules_sha256": np.array(sha(rules)), "n_rules": np.array([len(rules)]),
           "default_nh": np.array([default_nh], np.uint32)}
    for merge in (1, 0):
        st, m = ref.build_intervals(rules, default_nh, bool(merge))
        assert st == 0, ref.error()
        out[f"m_m{merge}"] = np.array([len(m.boundaries)])
        out[f"boundaries_sha256_m{merge}"] = np.array(sha(m.boundaries))
        out[f"next_hops_sha256_m{merge}"] = np.array(sha(m.next_hops))
        if merge:
            allk = sample_keys(rng, m.boundaries, n_interval // 4)
            keys = np.unique(rng.choice(allk, size=min(n_interval, len(allk)), replace=False))
            out["keys"] = keys
            out["interval_oracle"] = m.lookup(keys, 8)
            lk = np.unique(rng.choice(keys, size=min(n_linear, len(keys)), replace=False))
            out["linear_keys"] = lk
            out["linear_oracle"] = ref.linear_keys(rules, default_nh, lk, 8)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, len(rules), "rules ->", int(out["m_m1"][0]), "intervals,", len(out["keys"]), "keys,",
          len(out["linear_keys"]), "linear")


def main():
    ref = RefOracle()
    rng = np.random.default_rng(20260101)
    # {2001:db8::/32 -> 1, 2001:db8:1::/48 -> 2}
    spec = np.zeros(2, PREFIX_DTYPE)
    spec[0] = (0, 0x20010DB800000000, 32, 1, 0)
    spec[1] = (0, 0x20010DB800010000, 48, 2, 0)
    make(ref, "spec_two_rules", spec, 0, rng, 64)
    make(ref, "empty_fib", np.zeros(0, PREFIX_DTYPE), 5, rng, 64)
    for n, seed in ((10, 1), (1000, 2), (10000, 3)):
        make(ref, f"ref_synth_{n}", ref.synth_fib(n, seed, PREFIX_DTYPE), 0, rng)
    for n, dflt in ((300, True), (2000, False)):
        rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.5)
        make(ref, f"nested_{n}", rules, 9, rng)
    # SPEC S:486 acceptance size (10^5 rules) and the deepest tree (the 1M-prefix C2
    # FIB: depth 5 in the B200 layout, 16-bit next hops)
    for name, src in (("large_random_nested_100000", "random_nested:100000,100000"),
                      ("large_ref_synth_100000", "ref_synth:100000,4"),
                      ("large_workload_c2_fib", "workload:2")):
        rules, dflt = large_fixture_rules(src)
        make_large(ref, name, rules, dflt, rng, src)


if __name__ == "__main__":
    main()

"""Device-side FIB build (csrc/build.cu) vs the host build vs the reference.

The device build must produce the identical interval map (merge on and off) and
the identical line array, byte for byte, and refuse the same invalid rule sets
with the same Errc.
"""
import numpy as np
import pytest

from _util import MASK64, random_fib_rules, rules_array

pytestmark = pytest.mark.gpu


def _same_layout(lpm, fib):
    from paper_2604_14650_b200.gpu import device_lines
    host = lpm.build_tree(lpm.build_intervals(fib))
    dev = lpm.Fib.build_device(fib)
    assert dev.geometry == host.geometry
    np.testing.assert_array_equal(device_lines(dev), host.lines)
    return dev


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_device_build_workload_fibs(lpm, cuda, kind):
    from paper_2604_14650_b200.gpu import build_intervals_device
    fib = lpm.workload_fib(kind)
    for merge in (True, False):
        h = lpm.build_intervals(fib, merge_adjacent=merge)
        d = build_intervals_device(fib, merge_adjacent=merge)
        np.testing.assert_array_equal(d.boundaries, h.boundaries)
        np.testing.assert_array_equal(d.next_hops, h.next_hops)
    _same_layout(lpm, fib)


@pytest.mark.parametrize("n,dflt,vb", [(0, False, 1), (1, True, 1), (15, False, 1), (400, True, 2), (3000, False, 4),
                                       (30000, True, 2)])
def test_device_build_random_fibs(lpm, orc, cuda, n, dflt, vb):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    from paper_2604_14650_b200.gpu import build_intervals_device
    rng = np.random.default_rng(77 + n)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.5)
    top = {1: 255, 2: 65535, 4: 0xFFFFFFFE}[vb]
    rules["next_hop"] = rng.integers(1, top + 1, len(rules), dtype=np.uint64).astype(np.uint32)
    fib = lpm.FibTable(int(rng.integers(0, 100)), rules)
    st, ob, onh = orc.build_intervals(fib.rules, fib.default_next_hop)
    d = build_intervals_device(fib)
    np.testing.assert_array_equal(d.boundaries, ob)
    np.testing.assert_array_equal(d.next_hops, onh)
    _same_layout(lpm, fib)


def test_device_build_reference_fixtures(lpm, cuda):
    """The reference-generated golden fixtures (tests/golden) through the device build."""
    from pathlib import Path
    from paper_2604_14650_b200.gpu import build_intervals_device
    for f in sorted(p for p in (Path(__file__).resolve().parent / "golden").glob("*.npz")
                    if not p.stem.startswith("large_")):  # large ones: test_gpu_parity
        g = np.load(f)
        fib = lpm.FibTable(int(g["default_nh"][0]), g["rules"])
        for merge in (1, 0):
            d = build_intervals_device(fib, merge_adjacent=bool(merge))
            np.testing.assert_array_equal(d.boundaries, g[f"boundaries_m{merge}"])
            np.testing.assert_array_equal(d.next_hops, g[f"next_hops_m{merge}"])


def test_device_build_errors(lpm, cuda):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    A = 0x20010DB800000000
    cases = {
        "ReservedNextHop": [(A << 64, 32, 0xFFFFFFFF)],
        "SentinelCollision": [((MASK64 - 1) << 64, 64, 3)],
        "DuplicatePrefix": [(A << 64, 32, 1), (A << 64, 32, 2)],
        "UnsupportedPrefixLength": [(A << 64, 65, 1)],
        "InvalidArgument": [((A | 1) << 64, 32, 1)],
    }
    for code, rules in cases.items():
        fib = lpm.FibTable(0, rules_array(rules, PREFIX_DTYPE))
        for build in (lpm.build_intervals, lambda f: lpm.Fib.build_device(f)):
            with pytest.raises(lpm.Lpm6Error) as e:
                build(fib)
            assert e.value.code == code, (code, e.value)
    # the first offending rule in input order decides, as in the host build
    fib = lpm.FibTable(0, rules_array([(A << 64, 65, 1), (A << 64, 32, 0xFFFFFFFF)], PREFIX_DTYPE))
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.Fib.build_device(fib)
    assert e.value.code == "UnsupportedPrefixLength"


def test_device_built_fib_lookups(lpm, orc, cuda):
    """Lookups through a device-built C2 FIB equal the oracle on a 16M-query sample."""
    torch = cuda
    info = lpm.workload_info("C2")
    fib = lpm.workload_fib(info.fib_kind)
    dev = lpm.Fib.build_device(fib)
    gen = lpm.QueryGen("C2", fib)
    n = 1 << 24
    d = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    gen.run(0, n, d)
    out = dev.lookup_batch(d)
    st, b, nh = orc.build_intervals(fib.rules, fib.default_next_hop)
    want, _ = orc.lookup_batch(0, b, nh, d.cpu().numpy().view(np.uint64).reshape(-1, 2), threads=16)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint16).astype(np.uint32), want)

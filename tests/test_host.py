"""Host-side tests (no GPU): the C ABI library, the B200 layout, the workloads.

The layout is checked by walking it in numpy exactly as the kernel does (test
code only — the product has no CPU lookup) and comparing with the oracle.
"""
import ctypes as C
import os
import re
from pathlib import Path

import numpy as np
import pytest

from _util import MASK64, addrs_from_keys, boundary_probe_keys, random_fib_rules

ROOT = Path(__file__).resolve().parents[1]
LIB_DIR = ROOT / "paper_2604_14650_b200" / "lib"


# ---- the C ABI library -----------------------------------------------------------------------

def header_functions():
    text = (ROOT / "include" / "lpm6cu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lpm6(?:cu)?_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lpm):
    from paper_2604_14650_b200._lib import LIB_PATH, SIGNATURES
    names = header_functions()
    assert len(names) == len(SIGNATURES) == 62
    dll = C.CDLL(str(LIB_PATH))
    for name in names:
        assert hasattr(dll, name), f"{name} declared in include/lpm6cu.h but not exported"
        assert name in SIGNATURES, f"{name} has no ctypes binding"


def test_status_names_match_reference_errc(lpm):
    from paper_2604_14650_b200._lib import ERRC_NAMES, lib
    for i, name in enumerate(ERRC_NAMES, 1):
        assert lib().lpm6cu_status_name(i).decode() == name
    assert b"sm_100a" in lib().lpm6cu_version()


def test_no_cpu_fallback_without_gpu(lpm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    fib = lpm.workload_fib(0)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.Fib.build(fib)
    assert e.value.code == "CudaError"


# ---- the B200 layout --------------------------------------------------------------------------

def walk_layout(tree, keys):
    """Numpy restatement of the kernel's descent over the B200 layout (test-only)."""
    g = tree.geometry
    lines = tree.lines
    q = np.minimum(np.asarray(keys, np.uint64), np.uint64(MASK64 - 1))
    node = np.zeros(len(q), np.int64)
    for lvl in range(g.depth):
        base = g.level_start[lvl] + node * 16
        nd = lines[base[:, None] + np.arange(g.k)]
        node = node * g.b + (nd <= q[:, None]).sum(axis=1)
    base = g.level_start[g.depth] + node * g.leaf_words
    lf = lines[base[:, None] + np.arange(g.leaf_keys)]
    ordinal = (lf <= q[:, None]).sum(axis=1) - 1
    assert np.all(ordinal >= 0)
    return tree.leaf_values[node * g.leaf_keys + ordinal]


def check_layout(lpm, orc, fib, n_random=20000, seed=0, value_bytes=0, leaf_format=0):
    imap = lpm.build_intervals(fib)
    tree = lpm.build_tree(imap, value_bytes, leaf_format)
    g = tree.geometry
    m = len(imap)
    # leaves: 128-byte lines (kL = 14 / 12 / 8) or half lines of 6 keys + 2-byte next hops
    assert (g.leaf_words, g.leaf_keys) in ((16, {1: 14, 2: 12, 4: 8}[g.value_bytes]), (8, 6))
    if g.leaf_words == 8:
        assert g.value_bytes == 2 and g.leaf_image == 0
        lv = tree.lines[g.level_start[g.depth]: g.level_start[g.depth] + g.leaf_nodes * 8].reshape(-1, 8)
        vals = lv[:, 6:8].copy().view(np.uint16)[:, :6].reshape(-1)  # words 6-7: the six next hops
        np.testing.assert_array_equal(vals.astype(np.uint32), tree.leaf_values)
        assert g.image_start == g.level_start[g.depth] + g.leaf_nodes * 8
    # geometry: 15 separators + pad per internal line, arity 16; minimal depth; compact levels
    assert (g.k, g.b) == (15, 16)
    assert g.leaf_keys * 16 ** g.depth >= m and (g.depth == 0 or g.leaf_keys * 16 ** (g.depth - 1) < m)
    assert g.leaf_nodes == -(-m // g.leaf_keys)
    for lvl in range(g.depth):
        assert g.level_nodes[lvl] == -(-g.level_nodes[lvl + 1] // 16)
    assert g.level_nodes[0] == 1
    # leaves: boundaries then sentinels; values replicate the last one
    lk = tree.leaf_keys_array()
    np.testing.assert_array_equal(lk[:m], imap.boundaries)
    assert np.all(lk[m:] == np.uint64(MASK64))
    np.testing.assert_array_equal(tree.leaf_values[:m], imap.next_hops)
    assert np.all(tree.leaf_values[m:] == imap.next_hops[-1])
    # internal separators = boundary[(n*16 + j + 1) * span], word 15 = sentinel pad
    span = g.leaf_keys
    for lvl in range(g.depth - 1, -1, -1):
        nodes = g.level_nodes[lvl]
        idx = (np.arange(nodes)[:, None] * g.b + np.arange(g.k)[None, :] + 1) * span
        want = np.where(idx < m, imap.boundaries[np.minimum(idx, m - 1)], np.uint64(MASK64))
        got = tree.lines[g.level_start[lvl]: g.level_start[lvl] + nodes * 16].reshape(nodes, 16)
        np.testing.assert_array_equal(got[:, : g.k], want)
        assert np.all(got[:, 15] == np.uint64(MASK64))
        span *= g.b
    # the shared-memory image packs the 15 separators of internal levels [0, image_levels)
    assert g.image_levels <= g.depth
    for lvl in range(g.image_levels):
        nodes = g.level_nodes[lvl]
        src = tree.lines[g.level_start[lvl]: g.level_start[lvl] + nodes * 16].reshape(nodes, 16)
        off = g.image_start + g.level_start[lvl] // 16 * 15
        img = tree.lines[off: off + nodes * 15].reshape(nodes, 15)
        np.testing.assert_array_equal(img, src[:, :15])
    assert (g.total_words - g.image_start) * 8 <= 232448 - 1024
    # small trees: the leaf lines again at a 17-word stride after the internal image
    if g.leaf_image:
        assert g.image_levels == g.depth <= 3
        start = g.image_start + ((g.level_start[g.depth] // 16 * 15 * 8 + 15) // 16 * 16) // 8
        leaves = tree.lines[g.level_start[g.depth]: g.level_start[g.depth] + g.leaf_nodes * 16].reshape(-1, 16)
        img = tree.lines[start: start + g.leaf_nodes * 17].reshape(-1, 17)
        np.testing.assert_array_equal(img[:, :16], leaves)
        assert np.all(img[:, 16] == np.uint64(MASK64))
        assert g.total_words == start + (g.leaf_nodes * 17 * 8 + 15) // 16 * 16 // 8
    # the descent the kernel performs gives the oracle's answer
    rng = np.random.default_rng(seed)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, n_random, dtype=np.uint64)])
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(keys), threads=8)
    np.testing.assert_array_equal(walk_layout(tree, keys), want)
    return tree


@pytest.mark.parametrize("kind", [0, 1])
def test_layout_workload_fibs(lpm, orc, kind):
    tree = check_layout(lpm, orc, lpm.workload_fib(kind))
    assert tree.geometry.depth == {0: 2, 1: 4}[kind]
    assert tree.geometry.leaf_image == {0: 1, 1: 0}[kind]  # C0's whole tree fits shared memory


def test_half_leaf_layout_c2_auto(lpm, orc):
    """The 1M-prefix C2 FIB (2-byte next hops, a level in L2) gets half-line leaves by
    the automatic rule: the same depth (5) and the same four shared-memory levels."""
    tree = check_layout(lpm, orc, lpm.workload_fib(2), n_random=5000)
    g = tree.geometry
    assert g.leaf_words == 8 and g.leaf_keys == 6 and g.depth == 5 and g.image_levels == 4
    full = lpm.plan_layout(g.num_keys, 2, lpm.fib.LEAF_FULL)
    assert full.leaf_words == 16 and full.depth == g.depth and full.image_levels == g.image_levels
    # C1 (1-byte next hops, whole internal tree staged) keeps full lines
    assert lpm.plan_layout(387232, 1).leaf_words == 16
    with pytest.raises(lpm.Lpm6Error):
        lpm.plan_layout(1000, 1, lpm.fib.LEAF_HALF)  # half lines hold 2-byte next hops only


@pytest.mark.parametrize("n,dflt", [(0, False), (1, True), (13, False), (14, True), (300, False), (5000, True),
                                    (40000, True)])
def test_half_leaf_layout_forced(lpm, orc, n, dflt):
    """Half-line leaves forced on random FIBs with 2-byte next hops: the layout walk
    (the kernel's descent restated in numpy) matches the oracle on every boundary."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(n + 7)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.4)
    tree = check_layout(lpm, orc, lpm.FibTable(3, rules), n_random=3000, value_bytes=2,
                        leaf_format=lpm.fib.LEAF_HALF)
    assert tree.geometry.leaf_words == 8


@pytest.mark.parametrize("n,dflt", [(0, False), (1, True), (13, False), (14, True), (300, False), (5000, True)])
def test_layout_random_fibs(lpm, orc, n, dflt):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(n)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.4)
    rules["next_hop"] = rng.integers(1, 250, len(rules))
    check_layout(lpm, orc, lpm.FibTable(int(rng.integers(0, 9)), rules))


@pytest.mark.parametrize("vb,kl", [(1, 14), (2, 12), (4, 8)])
def test_layout_value_widths(lpm, vb, kl):
    b = np.arange(1000, dtype=np.uint64) * 977
    nh = (np.arange(1000) % 200 + 1).astype(np.uint32)
    imap = lpm.IntervalMap(b, nh, 0)
    t = lpm.build_tree(imap, vb)
    g = t.geometry
    assert g.value_bytes == vb and g.leaf_keys == kl
    leaves = t.lines[g.level_start[g.depth]: g.level_start[g.depth] + g.leaf_nodes * 16].reshape(-1, 16)
    raw = leaves.view(np.uint8).reshape(-1, 128)[:, kl * 8: kl * 8 + kl * vb]
    vals = raw.copy().view({1: np.uint8, 2: np.uint16, 4: np.uint32}[vb]).reshape(-1)
    np.testing.assert_array_equal(vals[:1000], nh)


def test_layout_value_width_errors(lpm):
    imap = lpm.IntervalMap(np.array([0, 5], np.uint64), np.array([1, 300], np.uint32), 0)
    assert lpm.build_tree(imap).geometry.value_bytes == 2
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.build_tree(imap, 1)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(lpm.Lpm6Error):
        lpm.build_tree(imap, 3)


def test_plan_layout_depths(lpm):
    for m, d in ((1, 0), (14, 0), (15, 1), (14 * 16, 1), (14 * 16 + 1, 2), (387232, 4)):
        assert lpm.plan_layout(m, 1).depth == d
    assert lpm.plan_layout(1893858, 2).depth == 5
    g = lpm.plan_layout(12 * 16 ** 6 + 1, 2)
    assert g.depth == 7


# ---- workloads ---------------------------------------------------------------------------------

def test_workload_fibs_match_baseline_configs(lpm):
    f0, f1 = lpm.workload_fib(0), lpm.workload_fib(1)
    assert len(f0) == 1001 and len(f1) == 200001          # + ::/0
    for f in (f0, f1):
        r = f.rules
        assert np.sum(r["length"] == 0) == 1
        assert r["next_hop"].min() >= 1 and r["next_hop"].max() <= 255
    r = f0.rules[f0.rules["length"] > 0]
    assert r["length"].min() >= 16 and r["length"].max() <= 64
    r = f1.rules[f1.rules["length"] > 0]
    agg = r[r["length"] <= 24]
    assert len(agg) >= 2000
    assert np.all((agg["value_hi"] >> np.uint64(61)) == 1)  # 2000::/3
    share48 = np.mean(r["length"] == 48)
    assert 0.40 < share48 < 0.48


def test_workload_c2_fib(lpm):
    f2 = lpm.workload_fib(2)
    r = f2.rules
    assert len(f2) == 1_000_000 and np.sum(r["length"] == 0) == 0
    assert r["next_hop"].max() > 255 and r["next_hop"].max() <= 65535
    assert lpm.build_tree(lpm.build_intervals(f2)).geometry.depth == 5


def test_query_generator(lpm):
    fib = lpm.workload_fib(1)
    a = lpm.workload_queries_host("C1", fib, 0, 200000)
    b = lpm.workload_queries_host("C1", fib, 100000, 100000)
    np.testing.assert_array_equal(a[100000:], b)          # counter-based: any slice regenerates exactly
    hi = a[:, 1]
    in2000 = (hi >> np.uint64(61)) == 1
    assert in2000.mean() > 0.95                              # 90% in-prefix (FIB is in 2000::/3) + 10% in 2000::/3
    u = lpm.workload_queries_host("C3a", fib, 0, 100000)
    assert 0.08 < ((u[:, 1] >> np.uint64(61)) == 1).mean() < 0.17   # uniform over 128 bits
    z = lpm.workload_queries_host("C3b", fib, 0, 100000)
    _, counts = np.unique(z[:, 1] >> np.uint64(16), return_counts=True)
    assert counts.max() > 1000                               # Zipf(1.1): heavy head


def test_ref_oracle_fixture_generator_is_reproducible(ref):
    """The golden fixtures regenerate bit-identically from the reference."""
    import subprocess
    import sys
    import tempfile
    src = ROOT / "tests" / "golden" / "make_golden.py"
    with tempfile.TemporaryDirectory() as d:
        code = src.read_text().replace('HERE = Path(__file__).resolve().parent', f'HERE = Path({str(src.parent)!r})')
        code = code.replace('np.savez_compressed(HERE / f"{name}.npz", **out)',
                            f'np.savez_compressed(Path({d!r}) / f"{{name}}.npz", **out)')
        p = Path(d) / "gen.py"
        p.write_text(code)
        subprocess.run([sys.executable, str(p)], check=True, capture_output=True)
        for f in (ROOT / "tests" / "golden").glob("*.npz"):
            a, b = np.load(f), np.load(Path(d) / f.name)
            for k in a.files:
                np.testing.assert_array_equal(a[k], b[k])


def test_reference_dropin_without_gpu():
    """A reference lpm6::FibTable handed to lpm6::gpu::Fib (oracle/ref_dropin_demo.cpp):
    the host build matches the reference; without a GPU the lookup refuses (no fallback)."""
    import subprocess
    import torch
    exe = ROOT / "oracle" / "_ref" / "ref_dropin_demo"
    if not exe.exists():
        pytest.skip("drop-in demo not built (reference sources absent at build time)")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_gpu_parity.py::test_reference_dropin")
    r = subprocess.run([str(exe), "3000", "20000", "--no-gpu-ok"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CudaError" in r.stdout


def test_missing_library_fails_loudly():
    """Without the built library the package refuses to run (no CPU fallback)."""
    import subprocess
    import sys
    code = ("import paper_2604_14650_b200 as lpm\n"
            "try:\n    lpm.workload_fib(0)\nexcept ImportError as e:\n    print('ImportError', e)\n")
    env = dict(os.environ, LPM6CU_LIB="/nonexistent/liblpm6cu.so")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert "ImportError" in r.stdout and "no CPU fallback" in r.stdout, r.stdout + r.stderr


def test_header_is_plain_c(tmp_path):
    """include/lpm6cu.h compiles as C99 and a C program links against the library."""
    import subprocess
    exe = tmp_path / "capi_demo"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
                        str(ROOT / "tests" / "c" / "capi_demo.c"), "-L", str(LIB_DIR), "-llpm6cu",
                        f"-Wl,-rpath,{LIB_DIR}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode in (0, 2), run.stdout + run.stderr  # 2: no GPU in this container


ABI_NULL_PROBE = r'''
import ctypes as C
from paper_2604_14650_b200._lib import SIGNATURES, lib
L = lib()
bad = []
for name, (res, args) in SIGNATURES.items():
    if res is not C.c_int:
        continue
    vals = [0 if a in (C.c_int, C.c_uint32, C.c_uint64) else None for a in args]
    st = getattr(L, name)(*vals)
    if st not in (0, 1, 2, 3, 6, 9, 10, 11, 12, 13, 14):
        bad.append((name, st))
print("ABI-OK" if not bad else bad)
'''


def run_abi_null_probe():
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", ABI_NULL_PROBE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ABI-OK" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])


def test_abi_rejects_null_arguments():
    """Every int-returning ABI entry point called with NULL / zero arguments returns
    a status (never crashes): run in a subprocess so a segfault fails the test."""
    run_abi_null_probe()

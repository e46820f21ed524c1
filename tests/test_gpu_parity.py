"""GPU parity: the sm_100a lookup (through the C ABI) vs the CPU oracle.

Every comparison is bit-exact. The oracle is the C restatement
(oracle/lpm6_oracle.c, pinned to the reference in test_oracle.py); where
oracle/_ref is present the reference's own lookup_interval_oracle is checked too.
"""
import numpy as np
import pytest

from _util import MASK64, addrs_from_keys, boundary_probe_keys, large_rules, random_fib_rules

pytestmark = pytest.mark.gpu

LANES = (4,)


def oracle_next_hops(orc, imap_b, imap_nh, addrs):
    out, _ = orc.lookup_batch(0, imap_b, imap_nh, addrs, threads=8)
    return out


def run_lookup(cuda, fib_dev, addrs_np):
    torch = cuda
    a = torch.from_numpy(addrs_np.view(np.uint8).reshape(-1, 16)).cuda()
    out = fib_dev.lookup_batch(a)
    torch.cuda.synchronize()
    return out.cpu().numpy().view({1: np.uint8, 2: np.uint16, 4: np.uint32}[out.element_size()])


def check_fib(lpm, orc, cuda, fib, addrs, lanes=LANES, smem_levels=(None, 0, 1, 2, 3, 4, 5, 6, 7), value_bytes=0,
              leaf_format=0):
    imap = lpm.build_intervals(fib)
    st, ob, onh = orc.build_intervals(fib.rules, fib.default_next_hop)
    assert st == 0
    np.testing.assert_array_equal(imap.boundaries, ob)
    np.testing.assert_array_equal(imap.next_hops, onh)
    want = oracle_next_hops(orc, ob, onh, addrs)
    dev = lpm.Fib.build(fib, value_bytes=value_bytes, leaf_format=leaf_format)
    for g in lanes:
        for t in smem_levels:
            geo = dev.geometry
            if t is not None and t > geo.depth + geo.leaf_image:  # depth + 1: leaf image (small trees)
                continue
            dev.set_kernel_config(lanes_per_query=g, smem_levels=t)
            for checked in (False, True):
                dev.set_checked(checked)
                if checked:
                    dev.node_visits(reset=True)
                got = run_lookup(cuda, dev, addrs).astype(np.uint32)
                bad = np.nonzero(got != want)[0]
                assert len(bad) == 0, (f"G={g} T={t} checked={checked}: {len(bad)} mismatches, first key "
                                       f"{int(addrs[bad[0], 1]):#x} want {want[bad[0]]} got {got[bad[0]]}")
                if checked:
                    assert dev.violations() == 0
                    # fixed node visits: depth + 1 lines per query whatever the split
                    assert dev.node_visits() == len(addrs) * (dev.geometry.depth + 1)
    dev.set_checked(False)
    return dev, want


def test_c0_full_workload(lpm, orc, cuda):
    """C0: 1,048,576 queries, whole-tree-in-smem and L2 variants, device query generator == host."""
    info = lpm.workload_info("C0")
    fib = lpm.workload_fib(info.fib_kind)
    addrs = lpm.workload_queries_host("C0", fib, 0, info.n_queries)
    torch = cuda
    gen = lpm.QueryGen("C0", fib)
    d = torch.empty((info.n_queries, 16), dtype=torch.uint8, device="cuda")
    gen.run(0, info.n_queries, d)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d.cpu().numpy().view(np.uint64).reshape(-1, 2), addrs)
    check_fib(lpm, orc, cuda, fib, addrs)


@pytest.mark.parametrize("n,with_default", [(0, False), (0, True), (1, False), (10, True), (1000, False),
                                            (10000, True), (100000, False)])
def test_random_fibs_boundaries(lpm, orc, cuda, n, with_default):
    """Random FIBs (depth 0..4): every boundary and boundary+-1, ::, all-ones, random and in-prefix keys."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(1000 + n)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, with_default)
    fib = lpm.FibTable(default_next_hop=int(rng.integers(0, 200)), rules=rules)
    imap = lpm.build_intervals(fib)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 20000, dtype=np.uint64)])
    if len(rules):
        pick = rules[rng.integers(0, len(rules), 20000)]
        ln = pick["length"].astype(np.uint64)
        keep = np.where(ln == 0, np.uint64(0), (~np.uint64(0)) << (np.uint64(64) - ln))
        keys = np.concatenate([keys, (pick["value_hi"] & keep) | (rng.integers(0, 2**64, 20000, dtype=np.uint64) & ~keep)])
    addrs = addrs_from_keys(keys, rng)
    check_fib(lpm, orc, cuda, fib, addrs)


@pytest.mark.parametrize("vb", [1, 2, 4])
def test_value_widths(lpm, orc, cuda, vb):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(vb)
    rules = random_fib_rules(rng, 3000, PREFIX_DTYPE, True)
    top = {1: 255, 2: 65535, 4: 0xFFFFFFFE}[vb]
    rules["next_hop"] = rng.integers(1, top + 1, len(rules), dtype=np.uint64).astype(np.uint32)
    fib = lpm.FibTable(7, rules)
    imap = lpm.build_intervals(fib)
    addrs = addrs_from_keys(np.concatenate([boundary_probe_keys(imap.boundaries),
                                            rng.integers(0, 2**64, 5000, dtype=np.uint64)]), rng)
    dev, _ = check_fib(lpm, orc, cuda, fib, addrs, smem_levels=(None, 0))
    assert dev.geometry.value_bytes == vb


def test_reference_oracle_agrees(lpm, orc, ref, cuda):
    """The compiled reference's lookup_interval_oracle on the same C1 sample."""
    info = lpm.workload_info("C1")
    fib = lpm.workload_fib(info.fib_kind)
    addrs = lpm.workload_queries_host("C1", fib, 0, 1 << 20)
    st, rmap = ref.build_intervals(fib.rules, fib.default_next_hop)
    assert st == 0
    want = rmap.lookup(addrs[:, 1], threads=8)
    dev = lpm.Fib.build(fib)
    got = run_lookup(cuda, dev, addrs)
    np.testing.assert_array_equal(got.astype(np.uint32), want)


def test_host_buffers_pipeline(lpm, orc, cuda):
    """lookup_batch with host (numpy) buffers: chunked H2D/lookup/D2H path."""
    info = lpm.workload_info("C1")
    fib = lpm.workload_fib(info.fib_kind)
    n = (1 << 24) + 12345  # > 2 staging chunks, ragged tail
    addrs = lpm.workload_queries_host("C1", fib, 5, n)
    imap = lpm.build_intervals(fib)
    want = oracle_next_hops(orc, imap.boundaries, imap.next_hops, addrs)
    dev = lpm.Fib.build(fib)
    got = dev.lookup_batch(addrs)
    np.testing.assert_array_equal(got.astype(np.uint32), want)


def test_corrupted_device_fib_is_detected(lpm, orc, cuda):
    """Fault injection: moving one leaf key on the device must surface as a parity failure."""
    torch = cuda
    info = lpm.workload_info("C0")
    fib = lpm.workload_fib(info.fib_kind)
    imap = lpm.build_intervals(fib)
    tree = lpm.build_tree(imap)
    g = tree.geometry
    lines = tree.lines.copy()
    slot = g.num_keys // 2
    word = g.level_start[g.depth] + (slot // g.leaf_keys) * 16 + slot % g.leaf_keys
    assert lines[word] == imap.boundaries[slot]
    lines[word] += np.uint64(1)  # the boundary moves one key to the right
    assert g.leaf_image  # C0 is small: its leaves also have a shared-memory image
    img_start = g.image_start + ((g.level_start[g.depth] // 16 * 15 * 8 + 15) // 16 * 16) // 8
    img_word = img_start + (slot // g.leaf_keys) * 17 + slot % g.leaf_keys
    assert lines[img_word] == imap.boundaries[slot]
    probe = addrs_from_keys(np.array([imap.boundaries[slot]], np.uint64))
    want = oracle_next_hops(orc, imap.boundaries, imap.next_hops, probe)
    # leaves read from L2 (smem_levels = depth): the corrupted line is detected
    dev = lpm.Fib.wrap_device(g, torch.from_numpy(lines.view(np.int64)).cuda(), 0)
    dev.set_kernel_config(smem_levels=g.depth)
    assert run_lookup(cuda, dev, probe).astype(np.uint32)[0] != want[0]
    # leaves read from the shared-memory leaf image: corrupting that copy is detected
    lines2 = tree.lines.copy()
    lines2[img_word] += np.uint64(1)
    dev2 = lpm.Fib.wrap_device(g, torch.from_numpy(lines2.view(np.int64)).cuda(), 0)
    assert dev2.kernel_config()["smem_levels"] == g.depth + 1
    assert run_lookup(cuda, dev2, probe).astype(np.uint32)[0] != want[0]
    ok = lpm.Fib.from_tree(tree)
    assert run_lookup(cuda, ok, probe).astype(np.uint32)[0] == want[0]


def test_checked_mode_flags_corrupted_tree(lpm, orc, cuda):
    """A tree whose root routes past the end of level 1 is caught (no out-of-bounds read)."""
    torch = cuda
    fib = lpm.workload_fib(1)
    tree = lpm.build_tree(lpm.build_intervals(fib))
    g = tree.geometry
    lines = tree.lines.copy()
    lines[0:15] = 0                                   # every root separator <= every query: rank 15
    img = g.image_start                               # and its shared-memory copy
    lines[img: img + 15] = 0
    dev = lpm.Fib.wrap_device(g, torch.from_numpy(lines.view(np.int64)).cuda(), 0)
    dev.set_checked(True)
    addrs = addrs_from_keys(np.arange(1, 4097, dtype=np.uint64) << np.uint64(50))
    for t in (None, 0):                               # shared-memory and L2 descents
        dev.set_kernel_config(smem_levels=t)
        run_lookup(cuda, dev, addrs)
        assert dev.violations() & 3
    good = lpm.Fib.from_tree(tree)
    good.set_checked(True)
    run_lookup(cuda, good, addrs)
    assert good.violations() == 0


LINE_PATHS = (0, 1, 2, 3, 4)  # lpm6cu_kernel_config.line_path: every plan the tuner can pick


def test_c1_full_size(lpm, orc, cuda):
    """C1 at BASELINE size: 268,435,456 queries, every one checked against the oracle,
    on every line path."""
    mism, checked = _check_chunks(lpm, orc, cuda, "C1", range(4), 1 << 26)
    assert checked == 1 << 28 and mism == 0


def _check_chunks(lpm, orc, cuda, workload, chunks, chunk):
    torch = cuda
    info = lpm.workload_info(workload)
    fib = lpm.workload_fib(info.fib_kind)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib)
    gen = lpm.QueryGen(workload, fib)
    d = torch.empty((chunk, 16), dtype=torch.uint8, device="cuda")
    vdt = {1: np.uint8, 2: np.uint16, 4: np.uint32}[info.value_bytes]
    mism = checked = 0
    for c in chunks:
        gen.run(c * chunk, chunk, d)
        host_addrs = d.cpu().numpy().view(np.uint64).reshape(-1, 2)
        want = oracle_next_hops(orc, imap.boundaries, imap.next_hops, host_addrs)
        for lp in LINE_PATHS:  # one oracle pass, every line path
            dev.set_kernel_config(line_path=lp)
            out = dev.lookup_batch(d)
            got = out.cpu().numpy().view(vdt).astype(np.uint32)
            mism += int(np.count_nonzero(got != want))
        checked += chunk
    return mism, checked


def test_c2_full_size(lpm, orc, cuda):
    """C2 at BASELINE size: 1,073,741,824 queries over the 1M-prefix FIB, every one checked
    on every line path."""
    mism, checked = _check_chunks(lpm, orc, cuda, "C2", range(16), 1 << 26)
    assert checked == 1 << 30 and mism == 0


@pytest.mark.parametrize("workload", ["C3a", "C3b"])
def test_c3_full_size(lpm, orc, cuda, workload):
    """C3a (uniform) / C3b (Zipf 1.1) over the C1 FIB: all 268,435,456 queries."""
    mism, checked = _check_chunks(lpm, orc, cuda, workload, range(4), 1 << 26)
    assert checked == 1 << 28 and mism == 0


def test_c4_chunks(lpm, orc, cuda):
    """C4: first, middle and last of the 128 64M-address chunks (each seeded by its index)."""
    mism, checked = _check_chunks(lpm, orc, cuda, "C4", [0, 63, 127], 1 << 26)
    assert mism == 0


def test_reference_dropin(cuda):
    """The reference's own FibTable -> lpm6::gpu::Fib -> compared with the reference's oracles."""
    import subprocess
    from pathlib import Path
    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ref_dropin_demo"
    if not exe.exists():
        pytest.skip("drop-in demo not built")
    r = subprocess.run([str(exe), "50000", "2000000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout
    # the store phase: per-op outcomes equal the reference FibTable mutators', 3 commits
    assert r.stdout.count("store: epoch") == 3 and "store: epoch 4" in r.stdout


def test_concurrent_lookups_on_many_streams(lpm, orc, cuda):
    """A FIB handle is immutable: lookups from several host threads on their own
    streams (device buffers) and the host-buffer pipeline at the same time all
    return the oracle's answers (the reference's contract)."""
    import threading
    torch = cuda
    fib = lpm.workload_fib(1)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib)
    rng = np.random.default_rng(9)
    addrs = addrs_from_keys(rng.integers(0, 2**64, 1 << 18, dtype=np.uint64), rng)
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    errors = []

    def device_worker():
        try:
            s = torch.cuda.Stream()
            for _ in range(20):
                out = dev.lookup_batch(da, stream=s)
                s.synchronize()
                assert np.array_equal(out.cpu().numpy().astype(np.uint32), want)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    def host_worker():
        try:
            for _ in range(5):
                out = dev.lookup_batch(addrs)
                assert np.array_equal(out.astype(np.uint32), want)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=device_worker) for _ in range(4)] + \
              [threading.Thread(target=host_worker) for _ in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_small_and_ragged_batches(lpm, orc, cuda):
    """Batch sizes around the 32-query tile and the 4-lane group, and n = 0."""
    torch = cuda
    fib = lpm.workload_fib(1)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib)
    rng = np.random.default_rng(11)
    addrs = addrs_from_keys(rng.integers(0, 2**64, 5000, dtype=np.uint64), rng)
    want = oracle_next_hops(orc, imap.boundaries, imap.next_hops, addrs)
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    for n in (1, 2, 3, 4, 5, 31, 32, 33, 127, 129, 1023, 4095, 5000):
        out = torch.full((n + 64,), 0xAB, dtype=torch.uint8, device="cuda")  # canary past the end
        dev.lookup_batch(da[:n], out[:n])
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        np.testing.assert_array_equal(o[:n].astype(np.uint32), want[:n], err_msg=f"n={n}")
        assert np.all(o[n:] == 0xAB), f"n={n}: wrote past the end"
    empty = torch.empty((0, 16), dtype=torch.uint8, device="cuda")
    dev.lookup_batch(empty, torch.empty(0, dtype=torch.uint8, device="cuda"))  # no launch, no error


def test_depth6_tree(lpm, orc, cuda):
    """A 16M-interval map (depth 6, the deepest a realistic FIB reaches) laid out on
    the device from intervals; lookups against the interval oracle, every smem split."""
    torch = cuda
    m = 16_000_000
    rng = np.random.default_rng(12)
    gaps = rng.integers(1, 1 << 30, m, dtype=np.uint64)
    b = np.cumsum(gaps, dtype=np.uint64)
    b[0] = 0
    nh = rng.integers(1, 250, m, dtype=np.uint32)
    nh[1:][nh[1:] == nh[:-1]] ^= 1  # merged map: adjacent next hops differ
    imap = lpm.IntervalMap(b, nh, 0)
    dev = lpm.Fib.from_intervals(imap)
    g = dev.geometry
    assert g.depth == 6
    keys = np.concatenate([b[rng.integers(0, m, 100000)], rng.integers(0, int(b[-1]) + (1 << 32), 100000,
                                                                        dtype=np.uint64)])
    keys = np.concatenate([keys, keys + np.uint64(1), keys - np.uint64(1)])
    addrs = addrs_from_keys(keys, rng)
    want = oracle_next_hops(orc, b, nh, addrs)
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    for t in range(g.image_levels + 1):
        dev.set_kernel_config(smem_levels=t)
        for checked in (False, True):
            dev.set_checked(checked)
            out = dev.lookup_batch(da)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy().astype(np.uint32), want, err_msg=f"T={t}")
            if checked:
                assert dev.violations() == 0


def test_golden_fixtures_on_gpu(lpm, cuda):
    """The reference-generated golden answers (tests/golden, make_golden.py): every
    fixture key looked up on the GPU equals the reference's own interval oracle and
    linear (brute-force) oracle, every kernel mode."""
    from pathlib import Path
    files = sorted(f for f in (Path(__file__).resolve().parent / "golden").glob("*.npz")
                   if not f.stem.startswith("large_"))
    assert files
    for f in files:
        d = np.load(f)
        fib = lpm.FibTable(int(d["default_nh"][0]), d["rules"])
        keys = d["keys"].astype(np.uint64)
        addrs = addrs_from_keys(keys, np.random.default_rng(0))
        dev = lpm.Fib.build(fib)
        geo = dev.geometry
        for t in [None] + list(range(geo.depth + geo.leaf_image + 1)):
            dev.set_kernel_config(smem_levels=t)
            got = run_lookup(cuda, dev, addrs).astype(np.uint32)
            np.testing.assert_array_equal(got, d["interval_oracle"], err_msg=f"{f.name} T={t}")
            np.testing.assert_array_equal(got, d["linear_oracle"], err_msg=f"{f.name} T={t}")


@pytest.mark.parametrize("n", [50, 5000, 50000])
def test_merge_on_off_same_answers(lpm, orc, cuda, n):
    """Adjacent-interval merge ON vs OFF (intervals.hpp:26-29): different maps,
    identical lookups on the GPU, both equal to the oracle."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(40 + n)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, True, nest_p=0.5)
    rules["next_hop"] = rng.integers(1, 4, len(rules))  # few next hops: many mergeable neighbours
    fib = lpm.FibTable(0, rules)
    on, off = lpm.build_intervals(fib, True), lpm.build_intervals(fib, False)
    assert len(off) > len(on)
    keys = np.concatenate([boundary_probe_keys(off.boundaries), rng.integers(0, 2**64, 20000, dtype=np.uint64)])
    addrs = addrs_from_keys(keys, rng)
    want = oracle_next_hops(orc, on.boundaries, on.next_hops, addrs)
    for merge in (True, False):
        dev = lpm.Fib.build(fib, merge_adjacent=merge)
        assert dev.geometry.num_keys == (len(on) if merge else len(off))
        np.testing.assert_array_equal(run_lookup(cuda, dev, addrs).astype(np.uint32), want)


def test_plain_c_caller(cuda, tmp_path):
    """tests/c/capi_demo.c — a C99 program using only include/lpm6cu.h — on the GPU."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2604_14650_b200" / "lib"
    exe = tmp_path / "capi_demo"
    r = subprocess.run(["gcc", "-std=c99", "-I", str(root / "include"), str(root / "tests" / "c" / "capi_demo.c"),
                        "-L", str(lib), "-llpm6cu", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0 and "capi_demo ok" in run.stdout, run.stdout + run.stderr


def test_abi_rejects_null_arguments_on_gpu(cuda):
    """The NULL/zero-argument probe of every ABI entry point with a device present
    (calls get past the device checks here)."""
    from test_host import run_abi_null_probe
    run_abi_null_probe()


def test_abi_valid_handles_null_buffers(lpm, cuda):
    """Valid FIB / store handles with NULL buffers and n > 0: every call returns a
    status, nothing crashes (subprocess)."""
    import subprocess
    import sys
    from pathlib import Path
    code = r'''
import ctypes as C
import paper_2604_14650_b200 as lpm
from paper_2604_14650_b200._lib import SIGNATURES, lib
L = lib()
fib = lpm.Fib.build(lpm.workload_fib(0))
store = lpm.FibStore(lpm.workload_fib(0))
snap = C.c_void_p()
assert L.lpm6cu_store_acquire(store._h, C.byref(snap)) == 0
handles = {"fib": fib._h, "store": store._h, "snapshot": snap}
firsts = {"lpm6cu_fib_": "fib", "lpm6cu_lookup_": "fib", "lpm6cu_search_batch": "fib", "lpm6cu_store_": "store",
          "lpm6cu_snapshot_": "snapshot"}
bad = []
for name, (res, args) in SIGNATURES.items():
    if res is not C.c_int or name in ("lpm6cu_store_destroy", "lpm6cu_store_release", "lpm6cu_fib_destroy"):
        continue
    kind = next((v for k, v in firsts.items() if name.startswith(k)), None)
    if kind is None or name in ("lpm6cu_fib_build", "lpm6cu_fib_build_device", "lpm6cu_fib_create",
                                "lpm6cu_fib_wrap_device", "lpm6cu_fib_adopt_device", "lpm6cu_fib_load_snapshot",
                                "lpm6cu_fib_build_from_intervals", "lpm6cu_store_create"):
        continue
    vals = [handles[kind]] + [5 if a in (C.c_int, C.c_uint32, C.c_uint64) else None for a in args[1:]]
    st = getattr(L, name)(*vals)
    if st not in (0, 9, 13):
        bad.append((name, st))
L.lpm6cu_store_release(snap, None)
print("ABI-OK" if not bad else bad)
'''
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ABI-OK" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.parametrize("name", ["large_random_nested_100000", "large_ref_synth_100000", "large_workload_c2_fib"])
def test_golden_large_fixtures_on_gpu(lpm, cuda, name):
    """The hash-pinned reference fixtures (SPEC S:486's 10^5 rules; the 1M-prefix C2 FIB,
    a depth-5 tree with 16-bit next hops): every sampled key's next hop from the GPU
    equals the reference's own lookup_interval_oracle and linear-oracle answers, at
    every smem_levels and on every line path, for the host-built and the device-built
    FIB."""
    from pathlib import Path
    d = np.load(Path(__file__).resolve().parent / "golden" / f"{name}.npz")
    rules, dflt = large_rules(d)
    fib = lpm.FibTable(dflt, rules)
    keys = d["keys"].astype(np.uint64)
    addrs = addrs_from_keys(keys, np.random.default_rng(1))
    pos = np.searchsorted(d["keys"], d["linear_keys"])
    for dev in (lpm.Fib.build(fib), lpm.Fib.build_device(fib, 0)):
        geo = dev.geometry
        if name == "large_workload_c2_fib":
            assert geo.depth == 5 and geo.value_bytes == 2
        for t in [None] + list(range(geo.depth + geo.leaf_image + 1)):
            for lp in (0, 1, 2, 3, 4):
                dev.set_kernel_config(smem_levels=t, line_path=lp)
                got = run_lookup(cuda, dev, addrs).astype(np.uint32)
                np.testing.assert_array_equal(got, d["interval_oracle"], err_msg=f"{name} T={t} lp={lp}")
                np.testing.assert_array_equal(got[pos], d["linear_oracle"], err_msg=f"{name} T={t} lp={lp}")
        dev.close()


def test_c2_against_reference_library(lpm, ref, cuda):
    """2^26 C2 queries (the 1M-prefix FIB, depth 5, 16-bit next hops) looked up on the
    GPU and by the reference's own build_intervals + lookup_interval_oracle
    (oracle/_ref, intervals.cpp:33-93,142-145), on every host thread."""
    import os
    torch = cuda
    info = lpm.workload_info("C2")
    fib = lpm.workload_fib(info.fib_kind)
    dev = lpm.Fib.build(fib)
    gen = lpm.QueryGen("C2", fib)
    n = 1 << 26
    d = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    gen.run(0, n, d)
    st, rmap = ref.build_intervals(fib.rules, fib.default_next_hop)
    assert st == 0
    keys = np.ascontiguousarray(d.cpu().numpy().view(np.uint64).reshape(-1, 2)[:, 1])
    want = rmap.lookup(keys, os.cpu_count() or 8)
    got = dev.lookup_batch(d).cpu().numpy().view(np.uint16).astype(np.uint32)
    assert int(np.count_nonzero(got != want)) == 0


@pytest.mark.slow
def test_c4_every_chunk(lpm, orc, cuda):
    """C4 in full: all 128 chunks of 64M queries (8,589,934,592 lookups) on the tuned
    line path, every next hop compared with the oracle (chunk c is seeded by c, so this
    is exactly the stream bench.py's C4 line and its output digest cover)."""
    import os
    torch = cuda
    info = lpm.workload_info("C4")
    fib = lpm.workload_fib(info.fib_kind)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib)
    gen = lpm.QueryGen("C4", fib)
    chunk = info.chunk
    d = torch.empty((chunk, 16), dtype=torch.uint8, device="cuda")
    gen.run(0, chunk, d)
    dev.tune_line_path(d)
    threads = os.cpu_count() or 8
    mism = 0
    for c in range(info.n_queries // chunk):
        gen.run(c * chunk, chunk, d)
        got = dev.lookup_batch(d).cpu().numpy().view(np.uint16).astype(np.uint32)
        host_addrs = d.cpu().numpy().view(np.uint64).reshape(-1, 2)
        want = oracle_next_hops_threads(orc, imap.boundaries, imap.next_hops, host_addrs, threads)
        mism += int(np.count_nonzero(got != want))
    assert mism == 0


def oracle_next_hops_threads(orc, b, nh, addrs, threads):
    out, _ = orc.lookup_batch(0, b, nh, addrs, threads=threads)
    return out


def test_kernel_smem_attribute_shared_across_fibs(lpm, orc, cuda):
    """FIBs of equal depth and next-hop width share one kernel, whose
    max-dynamic-shared-memory attribute used to be set to each FIB's own image size. A
    FIB with a smaller image (> 48 KB) resolving its plan then lowered it under a FIB
    with a larger one, whose later launches failed. Launch larger, smaller, larger."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(77)
    big = lpm.workload_fib(1)  # C1: depth 4, u8, 221 KB image
    rules = random_fib_rules(rng, 60000, PREFIX_DTYPE, True, nest_p=0.3)
    rules["next_hop"] = (rules["next_hop"] % 255) + 1  # u8 next hops like C1
    small = lpm.FibTable(0, rules)  # depth 4, 64 KB image
    db, ds = lpm.Fib.build(big), lpm.Fib.build(small)
    gb, gs = db.geometry, ds.geometry
    assert gb.depth == gs.depth and gb.value_bytes == gs.value_bytes == 1
    img = lambda dev: dev.kernel_config()["smem_levels"]
    keys = rng.integers(0, 2**64, 1 << 16, dtype=np.uint64)
    addrs = addrs_from_keys(keys, rng)
    wants = {}
    for name, fib in (("big", big), ("small", small)):
        st, b, nhs = orc.build_intervals(fib.rules, fib.default_next_hop)
        wants[name] = oracle_next_hops(orc, b, nhs, addrs)
    for name, dev in (("big", db), ("small", ds), ("big", db), ("small", ds), ("big", db)):
        got = run_lookup(cuda, dev, addrs).astype(np.uint32)
        np.testing.assert_array_equal(got, wants[name], err_msg=name)
    assert img(db) >= 1 and img(ds) >= 1


@pytest.mark.parametrize("n,dflt", [(1, True), (14, False), (3000, True), (60000, False)])
def test_half_leaf_fibs_every_mode(lpm, orc, cuda, n, dflt):
    """Half-line leaves (2-byte next hops, forced on random FIBs of every depth): every
    smem_levels setting, checked and unchecked (node visits = depth + 1), every line
    path, 8-byte keys and search_batch ordinals — all against the oracle."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    torch = cuda
    rng = np.random.default_rng(n + 11)
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, dflt, nest_p=0.4)
    fib = lpm.FibTable(5, rules)
    imap = lpm.build_intervals(fib)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 20000, dtype=np.uint64)])
    addrs = addrs_from_keys(keys, rng)
    dev, want = check_fib(lpm, orc, cuda, fib, addrs, value_bytes=2, leaf_format=2)
    assert dev.geometry.leaf_words == 8
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    dk = torch.from_numpy(np.ascontiguousarray(addrs[:, 1]).view(np.int64)).cuda()
    for lp in (0, 1, 2, 3):
        dev.set_kernel_config(line_path=lp)
        got = dev.lookup_batch(da).cpu().numpy().view(np.uint16).astype(np.uint32)
        gk = dev.lookup_keys(dk).cpu().numpy().view(np.uint16).astype(np.uint32)
        np.testing.assert_array_equal(got, want, err_msg=f"lp={lp}")
        np.testing.assert_array_equal(gk, want, err_msg=f"keys lp={lp}")
    ords, nh = dev.search_batch(dk)
    want_ord = np.searchsorted(imap.boundaries, np.minimum(keys, np.uint64(MASK64 - 1)), side="right") - 1
    np.testing.assert_array_equal(ords.cpu().numpy().astype(np.int64), want_ord)
    dev.close()


def test_half_leaf_device_build_matches_host(lpm, cuda):
    """The device build lays out half-line leaves bit-identically to the host build
    (forced on a random FIB; automatic on the 1M-prefix C2 FIB)."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rng = np.random.default_rng(5)
    fibs = [(lpm.FibTable(1, random_fib_rules(rng, 20000, PREFIX_DTYPE, True, nest_p=0.3)), 2),
            (lpm.workload_fib(2), 0)]
    from paper_2604_14650_b200.gpu import device_lines
    for fib, lf in fibs:
        host = lpm.build_tree(lpm.build_intervals(fib), 2, lf)
        devb = lpm.Fib.build_device(fib, 0, value_bytes=2, leaf_format=lf)
        assert host.geometry == devb.geometry and host.geometry.leaf_words == 8
        np.testing.assert_array_equal(device_lines(devb), host.lines)
        devb.close()

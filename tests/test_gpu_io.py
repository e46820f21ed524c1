"""Reference formats straight to the GPU, and the 8-byte-key lookup (search_batch's
input): PBT1 snapshot -> device FIB bit-identical to the rule-set build;
PBTR trace -> device keys -> lookups equal to the oracle."""
import numpy as np
import pytest

from _util import addrs_from_keys, boundary_probe_keys

pytestmark = pytest.mark.gpu

VDT = {1: np.uint8, 2: np.uint16, 4: np.uint32}


def device_lines(dev):
    import ctypes as C
    from paper_2604_14650_b200._lib import lib
    g = dev.geometry
    out = np.empty(g.total_words, np.uint64)
    assert lib().lpm6cu_fib_copy_lines(dev._h, out.ctypes.data, g.total_words) == 0
    return out


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_snapshot_to_device_equals_rule_build(lpm, cuda, kind, tmp_path):
    fib = lpm.workload_fib(kind)
    imap = lpm.build_intervals(fib)
    p = tmp_path / f"fib{kind}.pbt1"
    lpm.save_snapshot(imap, p)
    a = lpm.Fib.build(fib)
    b = lpm.Fib.load_snapshot(p)
    c = lpm.Fib.from_intervals(imap)
    assert a.geometry == b.geometry == c.geometry
    la = device_lines(a)
    np.testing.assert_array_equal(device_lines(b), la)
    np.testing.assert_array_equal(device_lines(c), la)


def test_snapshot_load_errors(lpm, cuda, tmp_path):
    p = tmp_path / "bad.pbt1"
    p.write_bytes(b"PBT1" + b"\0" * 30)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.Fib.load_snapshot(p)
    assert e.value.code == "BadSnapshotFile"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.Fib.load_snapshot(tmp_path / "missing.pbt1")
    assert e.value.code == "Io"
    with pytest.raises(lpm.Lpm6Error) as e:  # interval map contract on from_intervals
        lpm.Fib.from_intervals(lpm.IntervalMap(np.array([0, 5, 5], np.uint64), np.array([1, 2, 3], np.uint32), 0))
    assert e.value.code == "InvalidArgument"


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_lookup_keys_matches_oracle(lpm, orc, cuda, kind):
    torch = cuda
    fib = lpm.workload_fib(kind)
    imap = lpm.build_intervals(fib)
    rng = np.random.default_rng(kind)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 1 << 20, dtype=np.uint64)])
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(keys), threads=8)
    dev = lpm.Fib.build(fib)
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    for checked in (False, True):
        dev.set_checked(checked)
        out = dev.lookup_keys(dk)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(VDT[dev.geometry.value_bytes]).astype(np.uint32)
        np.testing.assert_array_equal(got, want)
        if checked:
            assert dev.violations() == 0
    # keys and addresses agree on the same stream of queries, for every staged-level split
    dev.set_checked(False)
    da = torch.from_numpy(addrs_from_keys(keys, rng).view(np.uint8).reshape(-1, 16)).cuda()
    for t in range(dev.geometry.depth + 1):
        dev.set_kernel_config(smem_levels=t)
        ok = dev.lookup_keys(dk)
        oa = dev.lookup_batch(da)
        torch.cuda.synchronize()
        assert torch.equal(ok, oa), t


def test_trace_to_device_and_lookup(lpm, orc, cuda, tmp_path):
    torch = cuda
    fib = lpm.workload_fib(1)
    imap = lpm.build_intervals(fib)
    info = lpm.workload_info("C1")
    n = (9 << 20) + 5  # > two 4M-key staging chunks, ragged tail
    addrs = lpm.workload_queries_host("C1", fib, 0, n)
    keys = addrs[:, 1].copy()
    p = tmp_path / "c1.pbtr"
    lpm.save_trace(keys, p)
    dk = lpm.load_trace(p)
    assert dk.numel() == n
    np.testing.assert_array_equal(dk.cpu().numpy().view(np.uint64), keys)
    dev = lpm.Fib.build(fib)
    out = dev.lookup_keys(dk)
    torch.cuda.synchronize()
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint8).astype(np.uint32), want)
    assert info.value_bytes == 1
    empty = tmp_path / "empty.pbtr"
    lpm.save_trace(np.zeros(0, np.uint64), empty)
    assert lpm.load_trace(empty).numel() == 0
    (tmp_path / "bad.pbtr").write_bytes(b"PBTR\x01\x00\x00\x00" + (5).to_bytes(8, "little") + b"\0" * 8)
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.load_trace(tmp_path / "bad.pbtr")
    assert e.value.code == "BadTraceFile"


def make_frames(addrs: np.ndarray, stride: int, dst_offset: int, rng) -> np.ndarray:
    """Frames with random bytes everywhere but the IPv6 destination field, written
    in network byte order (first hextet first) at dst_offset."""
    n = len(addrs)
    frames = rng.integers(0, 256, n * stride, dtype=np.uint8).reshape(n, stride)
    be = np.empty((n, 16), np.uint8)
    hi = addrs[:, 1].astype(">u8").view(np.uint8).reshape(n, 8)
    lo = addrs[:, 0].astype(">u8").view(np.uint8).reshape(n, 8)
    be[:, :8], be[:, 8:] = hi, lo
    frames[:, dst_offset:dst_offset + 16] = be
    return frames.reshape(-1)


@pytest.mark.parametrize("stride,off", [(64, 38), (80, 40), (72, 36), (66, 38), (65, 38), (128, 22), (64, 44), (48, 30), (72, 38), (68, 36)])
def test_lookup_packets_matches_oracle(lpm, orc, cuda, stride, off):
    """Packet ingest: the destination read straight from frames at every alignment
    (8/4/2/1) gives the oracle's next hops (Ethernet + IPv6: offset 38)."""
    torch = cuda
    fib = lpm.workload_fib(1)
    imap = lpm.build_intervals(fib)
    rng = np.random.default_rng(stride * 100 + off)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries)[:20000],
                           rng.integers(0, 2**64, 50000, dtype=np.uint64)])
    addrs = addrs_from_keys(keys, rng)
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    frames = torch.from_numpy(make_frames(addrs, stride, off, rng)).cuda()
    dev = lpm.Fib.build(fib)
    for checked in (False, True):
        dev.set_checked(checked)
        out = dev.lookup_packets(frames, len(addrs), stride, off)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy().astype(np.uint32), want)
    with pytest.raises(lpm.Lpm6Error):
        dev.lookup_packets(frames, len(addrs) + 1, stride, off)  # past the buffer


def test_single_process_nccl_replication(lpm, orc, cuda):
    """lpm6cu_fib_replicate: one grouped NCCL broadcast per call (here over the one
    visible GPU; the same call fans out to every device of a node)."""
    torch = cuda
    fib = lpm.workload_fib(1)
    src = lpm.Fib.build(fib)
    devices = list(range(torch.cuda.device_count()))
    reps = src.replicate(devices)
    assert len(reps) == len(devices)
    want_lines = device_lines(src)
    for r in reps:
        assert r.geometry == src.geometry
        np.testing.assert_array_equal(device_lines(r), want_lines)
    imap = lpm.build_intervals(fib)
    keys = np.random.default_rng(3).integers(0, 2**64, 1 << 16, dtype=np.uint64)
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(keys), threads=8)
    got = reps[0].lookup_keys(torch.from_numpy(keys.view(np.int64)).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy().astype(np.uint32), want)
    with pytest.raises(lpm.Lpm6Error) as e:
        src.replicate([len(devices)])  # devices[0] must be the source device
    assert e.value.code in ("InvalidArgument", "CudaError")


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_search_batch_ordinals(lpm, orc, cuda, kind):
    """search_batch: the interval ordinal of every key is the oracle's
    upper_bound - 1 (intervals.cpp:142-145), and the next hops match; ordinals-only
    mode writes no next hops."""
    torch = cuda
    fib = lpm.workload_fib(kind)
    imap = lpm.build_intervals(fib)
    rng = np.random.default_rng(20 + kind)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 1 << 18, dtype=np.uint64)])
    clamped = np.minimum(keys, np.uint64(2**64 - 2))
    want_ord = np.searchsorted(imap.boundaries, clamped, side="right") - 1
    want_nh, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(keys), threads=8)
    dev = lpm.Fib.build(fib)
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    for checked in (False, True):
        dev.set_checked(checked)
        ords, nhs = dev.search_batch(dk)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ords.cpu().numpy().astype(np.int64), want_ord)
        np.testing.assert_array_equal(nhs.cpu().numpy().view(VDT[dev.geometry.value_bytes]).astype(np.uint32),
                                      want_nh)
        assert np.array_equal(imap.next_hops[want_ord], want_nh)
    dev.set_checked(False)
    ords, nhs = dev.search_batch(dk, with_next_hops=False)
    torch.cuda.synchronize()
    assert nhs is None
    np.testing.assert_array_equal(ords.cpu().numpy().astype(np.int64), want_ord)


def test_lookup_keys_host_buffers(lpm, orc, cuda):
    """lookup_keys with numpy (host) buffers: the pipelined path with 8-byte keys."""
    fib = lpm.workload_fib(1)
    imap = lpm.build_intervals(fib)
    rng = np.random.default_rng(31)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries),
                           rng.integers(0, 2**64, (1 << 24) + 777, dtype=np.uint64)])  # > 2 chunks, ragged
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(keys), threads=8)
    dev = lpm.Fib.build(fib)
    got = dev.lookup_keys(keys)
    np.testing.assert_array_equal(got.astype(np.uint32), want)

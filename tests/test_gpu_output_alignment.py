"""Result buffers at any byte offset: the C ABI takes a plain `void* out`, so a
caller may pass an unaligned pointer (a slice of a byte buffer). The kernels
store next hops no wider than the buffer's alignment allows, never write outside
[out, out + n * value_bytes), and give the oracle's answers at every offset, for
every input format and for the shared-memory leaf image as well as L2 leaves;
the same holds for page-locked host buffers (zero-copy up to 2^20 queries)."""
import numpy as np
import pytest

from _util import addrs_from_keys, boundary_probe_keys, random_fib_rules

pytestmark = pytest.mark.gpu

CANARY = 0xA5


def _fib(lpm, rng, n, vb):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rules = random_fib_rules(rng, n, PREFIX_DTYPE, True, nest_p=0.3)
    rules["next_hop"] = rng.integers(1, (1 << (8 * vb)) - 1, len(rules), dtype=np.uint64).astype(np.uint32)
    return lpm.FibTable(int(rng.integers(1, 200)), rules)


@pytest.mark.parametrize("vb", [1, 2, 4])
@pytest.mark.parametrize("n_rules", [300, 40000])  # leaf image / leaves from L2
def test_any_output_offset(lpm, orc, cuda, vb, n_rules):
    torch = cuda
    rng = np.random.default_rng(vb * 100 + n_rules)
    fib = _fib(lpm, rng, n_rules, vb)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib, value_bytes=vb)
    assert dev.value_bytes == vb
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 5003, dtype=np.uint64)])
    n = len(keys)
    addrs = addrs_from_keys(keys, rng)
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    frames = torch.zeros((n, 64), dtype=torch.uint8, device="cuda")  # Ethernet + IPv6, destination at 38
    dst = np.zeros((n, 16), np.uint8)
    dst[:, :8] = keys.astype(">u8").view(np.uint8).reshape(-1, 8)  # network byte order
    frames[:, 38:54] = torch.from_numpy(dst).cuda()
    line_paths = (0, 2) if dev.geometry.leaf_image == 0 else (0,)
    for lp in line_paths:
        dev.set_kernel_config(line_path=lp)
        for off in range(0, 17):
            for mode in ("addr", "keys", "packets"):
                buf = torch.full((n * vb + 48,), CANARY, dtype=torch.uint8, device="cuda")
                out = buf[off: off + n * vb]
                if mode == "addr":
                    dev.lookup_batch(da, out)
                elif mode == "keys":
                    dev.lookup_keys(dk, out)
                else:
                    dev.lookup_packets(frames, n, 64, 38, out)
                torch.cuda.synchronize()
                b = buf.cpu().numpy()
                got = b[off: off + n * vb].copy().view({1: "<u1", 2: "<u2", 4: "<u4"}[vb]).astype(np.uint32)
                np.testing.assert_array_equal(got, want, err_msg=f"vb={vb} off={off} mode={mode} lp={lp}")
                assert (b[:off] == CANARY).all() and (b[off + n * vb:] == CANARY).all(), (vb, off, mode, lp)


@pytest.mark.parametrize("n", [1, 31, 4097, 65536, 1 << 20, (1 << 20) + 1])
def test_pinned_host_batches(lpm, orc, cuda, n):
    """Host buffers in page-locked memory: up to 2^20 queries go zero-copy (the kernel
    reads addresses and writes next hops over PCIe), larger batches through the copy
    pipeline; both give the oracle's answers, also into a result buffer at an odd
    offset, and pageable buffers keep working."""
    torch = cuda
    rng = np.random.default_rng(n)
    fib = _fib(lpm, rng, 20000, 2)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib, value_bytes=2)
    keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, n, dtype=np.uint64)])[:n]
    addrs = addrs_from_keys(keys, rng)
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    ha = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).pin_memory()
    hk = torch.from_numpy(keys.view(np.int64)).pin_memory()
    for off in (0, 1):
        buf = torch.full((2 * n + 16,), CANARY, dtype=torch.uint8).pin_memory()
        out = buf[off: off + 2 * n]
        dev.lookup_batch(ha.numpy(), out.numpy())
        got = buf.numpy()[off: off + 2 * n].copy().view("<u2").astype(np.uint32)
        np.testing.assert_array_equal(got, want, err_msg=f"n={n} off={off}")
        assert (buf.numpy()[:off] == CANARY).all() and (buf.numpy()[off + 2 * n:] == CANARY).all()
        buf.fill_(CANARY)
        dev.lookup_keys(hk.numpy(), out.numpy())
        got = buf.numpy()[off: off + 2 * n].copy().view("<u2").astype(np.uint32)
        np.testing.assert_array_equal(got, want, err_msg=f"keys n={n} off={off}")
    pageable = dev.lookup_batch(np.ascontiguousarray(addrs))  # numpy, not page-locked
    np.testing.assert_array_equal(pageable.astype(np.uint32), want)

"""Line paths (lpm6cu_kernel_config.line_path: which L1TEX pipe carries the leaf
and internal L2 lines), the tiles per warp of the texture leaf paths
(queries_per_lane 1, 2 or 4 at 1024 threads), the split-plane descent of the staged
levels (plane_levels) and the measured choice between them
(lpm6cu_fib_tune_line_path).

A line path changes only how a line reaches registers, so every answer must
equal the oracle's on every path; the tuner must leave the kernel config on one
of the paths and never change results."""
import numpy as np
import pytest

from _util import addrs_from_keys, boundary_probe_keys

pytestmark = pytest.mark.gpu

VIEW = {1: np.uint8, 2: np.uint16, 4: np.uint32}


@pytest.mark.parametrize("workload", ["C1", "C2", "C3b"])
def test_texture_line_path_matches_oracle_on_workloads(lpm, orc, cuda, workload):
    """2^22 queries of each workload plus every boundary ±1, every line path, address
    and key input: bit-exact against the oracle."""
    torch = cuda
    info = lpm.workload_info(workload)
    fib = lpm.workload_fib(info.fib_kind)
    imap = lpm.build_intervals(fib)
    dev = lpm.Fib.build(fib)
    gen = lpm.QueryGen(workload, fib)
    n = 1 << 22
    d = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    gen.run(0, n, d)
    torch.cuda.synchronize()
    host = d.cpu().numpy().view(np.uint64).reshape(-1, 2)
    probes = addrs_from_keys(boundary_probe_keys(imap.boundaries), np.random.default_rng(7))
    addrs = np.concatenate([host, probes])
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
    da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
    dk = torch.from_numpy(np.ascontiguousarray(addrs[:, 1]).view(np.int64)).cuda()
    view = VIEW[dev.geometry.value_bytes]
    for lp in (1, 2, 3, 4, 0):
        cfg = dev.set_kernel_config(line_path=lp)
        assert cfg["line_path"] == lp
        got = dev.lookup_batch(da)
        gk = dev.lookup_keys(dk)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy().view(view).astype(np.uint32), want, err_msg=f"lp={lp}")
        np.testing.assert_array_equal(gk.cpu().numpy().view(view).astype(np.uint32), want, err_msg=f"keys lp={lp}")
    # 2 and 4 tiles per warp (Phase A over all tiles, Phase B one tile at a time): the
    # texture leaf paths run them, the others fall back to one tile; results unchanged
    for qpl in (2, 4):
        for lp in (1, 4, 0, 2, 3):
            cfg = dev.set_kernel_config(line_path=lp, threads_per_cta=1024, queries_per_lane=qpl)
            assert cfg["queries_per_lane"] == qpl and cfg["line_path"] == lp
            # ragged batch: not a multiple of the 32 * qpl queries a warp takes per iteration
            m = len(da) - 77
            got = dev.lookup_batch(da[:m])
            gk = dev.lookup_keys(dk)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(got.cpu().numpy().view(view).astype(np.uint32), want[:m],
                                          err_msg=f"qpl={qpl} lp={lp}")
            np.testing.assert_array_equal(gk.cpu().numpy().view(view).astype(np.uint32), want,
                                          err_msg=f"keys qpl={qpl} lp={lp}")


    # split-plane descent of the staged levels (plane_levels P: levels 1 .. P - 1 as high /
    # low word planes, the rest packed), every P, on the shapes that run it and on those
    # that ignore it; smem_levels one below the depth as well (C2's other static staging)
    depth = dev.geometry.depth
    for t in (None, depth - 1):
        for pu in range(2, depth + 2):
            for qpl, lp in ((2, 1), (4, 1), (2, 4), (4, 4), (1, 1), (2, 2)):
                cfg = dev.set_kernel_config(smem_levels=t, line_path=lp, threads_per_cta=1024, queries_per_lane=qpl,
                                            plane_levels=pu)
                # kernels exist for P = 2, 3 and every staged level (reported as smem_levels)
                assert cfg["plane_levels"] == (cfg["smem_levels"] if pu >= cfg["smem_levels"] else min(pu, 3))
                m = len(da) - 77
                got = dev.lookup_batch(da[:m])
                torch.cuda.synchronize()
                np.testing.assert_array_equal(got.cpu().numpy().view(view).astype(np.uint32), want[:m],
                                              err_msg=f"planes {pu} smem_levels {t} qpl={qpl} lp={lp}")
    assert dev.set_kernel_config(plane_levels=1)["plane_levels"] == 0  # no plane level: packed


def test_tuner_picks_a_path_and_keeps_results(lpm, orc, cuda):
    torch = cuda
    for workload in ("C1", "C2", "C3b"):
        info = lpm.workload_info(workload)
        fib = lpm.workload_fib(info.fib_kind)
        dev = lpm.Fib.build(fib)
        gen = lpm.QueryGen(workload, fib)
        n = 1 << 24
        d = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
        gen.run(0, n, d)
        base = dev.lookup_batch(d).clone()
        chosen = dev.tune_line_path(d)
        assert chosen in (0, 1, 2, 3, 4)
        cfg = dev.kernel_config()
        assert cfg["line_path"] == chosen
        # the tuner also picks the tiles per warp: 2 or 4 only on the texture leaf paths
        assert cfg["queries_per_lane"] in ((1, 2, 4) if chosen in (1, 4) else (1,))
        # ... and the plane levels of the split-plane descent, only with 2 or 4 tiles
        assert cfg["plane_levels"] == 0 or (cfg["queries_per_lane"] > 1 and 2 <= cfg["plane_levels"] <= cfg["smem_levels"])
        again = dev.lookup_batch(d)
        torch.cuda.synchronize()
        assert torch.equal(base, again)


def test_tuner_on_checked_and_leaf_image_fibs_stays_on_lsu(lpm, cuda):
    """No texture leaf kernel exists for checked mode or the shared-memory leaf image:
    the tuner reports the LSU path, and lookups keep working."""
    torch = cuda
    fib = lpm.workload_fib(lpm.workload_info("C0").fib_kind)  # leaf-image tree
    dev = lpm.Fib.build(fib)
    a = torch.zeros((4096, 16), dtype=torch.uint8, device="cuda")
    assert dev.tune_line_path(a) == 0
    big = lpm.Fib.build(lpm.workload_fib(1))
    big.set_checked(True)
    assert big.tune_line_path(a) == 0
    big.lookup_batch(a)
    torch.cuda.synchronize()
    assert big.violations() == 0
    big.set_checked(False)


def test_line_path_argument_errors(lpm, cuda):
    torch = cuda
    dev = lpm.Fib.build(lpm.workload_fib(1))
    with pytest.raises(lpm.Lpm6Error):
        dev.set_kernel_config(line_path=5)
    with pytest.raises(lpm.Lpm6Error):
        dev.tune_line_path(np.zeros((16, 16), np.uint8))  # host buffers
    with pytest.raises(lpm.Lpm6Error):
        dev.tune_line_path(torch.zeros((0, 16), dtype=torch.uint8, device="cuda"))

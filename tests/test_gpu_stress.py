"""Randomised parity stress: random FIBs (0–60,000 rules, nesting, minimum
lengths, default route on/off, merge on/off, 1/2/4-byte next hops, host or
device build) through every kernel mode the FIB admits — every shared-memory
split incl. the leaf image, every line path and tile count, checked and unchecked, address / key /
search_batch inputs — against the CPU oracle on every boundary ±1 and random keys."""
import os

import numpy as np
import pytest

from _util import addrs_from_keys, boundary_probe_keys, random_fib_rules

pytestmark = pytest.mark.gpu


def test_random_fibs_every_mode(lpm, orc, cuda):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    torch = cuda
    # LPM6_STRESS_SEED / LPM6_STRESS_ITERS: longer soak runs with other seeds
    # (tools/gpu/run37.sh; the default is what the test suite runs).
    rng = np.random.default_rng(int(os.environ.get("LPM6_STRESS_SEED", "12345")))
    failures = []
    for it in range(int(os.environ.get("LPM6_STRESS_ITERS", "60"))):
        n = int(rng.choice([0, 1, 5, 50, 500, 5000, 20000, 60000]))
        rules = random_fib_rules(rng, n, PREFIX_DTYPE, bool(rng.integers(0, 2)), nest_p=float(rng.uniform(0, 0.7)),
                                 min_len=int(rng.integers(0, 40)))
        top = int(rng.choice([255, 65535, 0xFFFFFFFE]))
        if len(rules):
            rules["next_hop"] = rng.integers(1, top + 1, len(rules), dtype=np.uint64).astype(np.uint32)
        fib = lpm.FibTable(int(rng.integers(0, 255)), rules)
        merge = bool(rng.integers(0, 2))
        imap = lpm.build_intervals(fib, merge)
        keys = np.concatenate([boundary_probe_keys(imap.boundaries), rng.integers(0, 2**64, 20000, dtype=np.uint64)])
        addrs = addrs_from_keys(keys, rng)
        want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs, threads=8)
        dev = (lpm.Fib.build_device if it % 2 else lpm.Fib.build)(fib, merge_adjacent=merge)
        g = dev.geometry
        da = torch.from_numpy(addrs.view(np.uint8).reshape(-1, 16)).cuda()
        dk = torch.from_numpy(keys.view(np.int64)).cuda()
        view = {1: np.uint8, 2: np.uint16, 4: np.uint32}[g.value_bytes]
        for t in [None] + list(range(g.depth + g.leaf_image + 1)):
            # line paths (which L1TEX pipe carries the L2 lines) x tiles per warp (2 and 4
            # exist on the texture leaf paths 1 and 4)
            # ... x split-plane descent (plane_levels; runs on the 2- and 4-tile kernels)
            for lp, qpl, pu in ((0, 1, 0), (1, 1, 0), (2, 1, 0), (3, 1, 0), (4, 1, 0), (1, 2, 0), (1, 4, 0), (4, 2, 0),
                                (4, 4, 0), (1, 2, 2), (1, 4, 3), (4, 2, 8), (1, 4, 8), (4, 4, 2), (1, 1, 3)):
                dev.set_kernel_config(smem_levels=t, line_path=lp, threads_per_cta=1024, queries_per_lane=qpl,
                                      plane_levels=pu)
                for checked in (False, True):
                    dev.set_checked(checked)
                    for mode, got in (("addr", dev.lookup_batch(da)), ("keys", dev.lookup_keys(dk)),
                                      ("search", dev.search_batch(dk)[1])):
                        torch.cuda.synchronize()
                        if not np.array_equal(got.cpu().numpy().view(view).astype(np.uint32), want):
                            failures.append((it, n, t, lp, qpl, pu, checked, mode, g.depth, g.value_bytes))
                    if checked and dev.violations():
                        failures.append((it, "violations"))
        dev.set_checked(False)
    assert not failures, failures[:10]

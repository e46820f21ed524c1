"""Property-based GPU parity (hypothesis): generated FIBs and keys through every
kernel mode the FIB admits (shared-memory splits, leaf image, checked mode, key
input, search_batch ordinals) against the CPU oracle."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from _util import addrs_from_keys, boundary_probe_keys, rules_array
from test_properties import fibs

pytestmark = pytest.mark.gpu
MASK64 = (1 << 64) - 1


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(fibs(max_rules=300), st.lists(st.integers(0, MASK64), min_size=1, max_size=200), st.sampled_from([0, 1, 2, 4]))
def test_gpu_matches_oracle_on_generated_fibs(lpm, orc, cuda, fib_def, keys, vb):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    torch = cuda
    rules, dflt = fib_def
    fib = lpm.FibTable(dflt, rules_array(rules, PREFIX_DTYPE))
    imap = lpm.build_intervals(fib)
    need = 1 if imap.next_hops.max() <= 255 else 2
    vb = max(vb, need) if vb else 0
    k = np.concatenate([np.array(keys, np.uint64), boundary_probe_keys(imap.boundaries)])
    want, _ = orc.lookup_batch(0, imap.boundaries, imap.next_hops, addrs_from_keys(k), threads=1)
    want_ord = np.searchsorted(imap.boundaries, np.minimum(k, np.uint64(MASK64 - 1)), side="right") - 1
    dev = lpm.Fib.build(fib, value_bytes=vb)
    g = dev.geometry
    da = torch.from_numpy(addrs_from_keys(k).view(np.uint8).reshape(-1, 16)).cuda()
    dk = torch.from_numpy(k.view(np.int64)).cuda()
    view = {1: np.uint8, 2: np.uint16, 4: np.uint32}[g.value_bytes]
    for t, lp in [(t, lp) for t in [None] + list(range(g.depth + g.leaf_image + 1)) for lp in (0, 1, 2, 3, 4)]:
        dev.set_kernel_config(smem_levels=t, line_path=lp)
        for checked in (False, True):
            dev.set_checked(checked)
            out = dev.lookup_batch(da)
            ko = dev.lookup_keys(dk)
            ords, nhs = dev.search_batch(dk)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy().view(view).astype(np.uint32), want)
            np.testing.assert_array_equal(ko.cpu().numpy().view(view).astype(np.uint32), want)
            np.testing.assert_array_equal(ords.cpu().numpy().astype(np.int64), want_ord)
            np.testing.assert_array_equal(nhs.cpu().numpy().view(view).astype(np.uint32), want)
            if checked:
                assert dev.violations() == 0
    dev.set_checked(False)

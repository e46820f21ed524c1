"""A loose throughput floor on the bench's kernels: catches a catastrophic
regression (a wrong kernel picked, a spill storm, a lost shared-memory image)
without being sensitive to the box. Bench values are ~77 (C1) and ~58 (C2)
G lookups/s; the floors are about half of that."""
import pytest

pytestmark = pytest.mark.gpu

FLOORS = {"C1": 40.0, "C2": 30.0}


@pytest.mark.parametrize("workload", sorted(FLOORS))
def test_throughput_floor(lpm, cuda, workload):
    torch = cuda
    info = lpm.workload_info(workload)
    fib = lpm.workload_fib(info.fib_kind)
    dev = lpm.Fib.build(fib)
    n = 1 << 26
    d = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    lpm.QueryGen(workload, fib).run(0, n, d)
    out = torch.empty(n * info.value_bytes, dtype=torch.uint8, device="cuda")
    dev.tune_line_path(d, out)
    for _ in range(3):
        dev.lookup_batch(d, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dev.lookup_batch(d, out)
    e1.record()
    torch.cuda.synchronize()
    glps = 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    assert glps >= FLOORS[workload], f"{workload}: {glps:.1f} G lookups/s"

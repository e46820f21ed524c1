"""Time the GPU FIB build (and the host build) for the workload FIBs."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2604_14650_b200 as lpm  # noqa: E402

for kind in (1, 2):
    fib = lpm.workload_fib(kind)
    t0 = time.perf_counter()
    lpm.build_tree(lpm.build_intervals(fib))
    host = (time.perf_counter() - t0) * 1e3
    lpm.Fib.build_device(fib).close()
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lpm.Fib.build_device(fib).close()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    print(f"fib_kind {kind}: {len(fib)} rules  host build {host:.1f} ms  device build {best:.2f} ms")

"""Call-to-result latency of small pinned host batches (zero-copy path) on the C1 FIB
for each number of shared-memory levels: what staging the image costs a tiny batch."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2604_14650_b200 as lpm
from paper_2604_14650_b200._lib import lib
fib = lpm.workload_fib(1); dev = lpm.Fib.build(fib)
gen = lpm.QueryGen("C1", fib)
d = torch.empty((1 << 16, 16), dtype=torch.uint8, device="cuda"); gen.run(0, 1 << 16, d); torch.cuda.synchronize()
fn = lib().lpm6cu_lookup_batch
for b in (32, 256, 4096, 65536):
    ha = d[:b].cpu().pin_memory().numpy(); ho = torch.empty(b, dtype=torch.uint8).pin_memory().numpy()
    row = {}
    for t in (4, 3, 2, 1, 0):
        dev.set_kernel_config(smem_levels=t)
        for _ in range(20): fn(dev._h, ha.ctypes.data, b, ho.ctypes.data, None)
        lat = []
        for _ in range(300):
            t0 = time.perf_counter(); fn(dev._h, ha.ctypes.data, b, ho.ctypes.data, None); lat.append((time.perf_counter() - t0) * 1e6)
        row[t] = round(float(np.median(lat)), 1)
    # device-side kernel time alone (device buffers, events)
    print(b, row)

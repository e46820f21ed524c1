"""Call-to-result latency of lpm6cu_lookup_batch on host buffers (page-locked vs pageable), C1 FIB;
batch sizes from argv."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2604_14650_b200 as lpm
fib = lpm.workload_fib(1); dev = lpm.Fib.build(fib)
gen = lpm.QueryGen("C1", fib)
sizes = [int(x) for x in (sys.argv[1:] or ["256", "4096", "16384", "65536"])]
nmax = max(sizes)
d = torch.empty((nmax, 16), dtype=torch.uint8, device="cuda"); gen.run(0, nmax, d); torch.cuda.synchronize()
import ctypes as C
from paper_2604_14650_b200._lib import lib
for b in sizes:
    ha = d[:b].cpu().pin_memory(); ho = torch.empty(b, dtype=torch.uint8).pin_memory()
    hp = d[:b].cpu().numpy().copy(); hpo = np.empty(b, np.uint8)
    res = {}
    for name, a, o in (("pinned", ha.numpy(), ho.numpy()), ("pageable", hp, hpo)):
        for _ in range(20): dev.lookup_batch(a, o)
        # direct ctypes call to strip Python wrapper overhead
        fn = lib().lpm6cu_lookup_batch
        ap, op = a.ctypes.data, o.ctypes.data
        lat = []
        for _ in range(300):
            t0 = time.perf_counter(); fn(dev._h, ap, b, op, None); lat.append((time.perf_counter() - t0) * 1e6)
        res[name] = round(float(np.median(lat)), 1)
    print(b, res)

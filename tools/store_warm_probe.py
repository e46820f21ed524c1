"""Store first-commit probe: the test_first_commit_is_warm sequence in a plain process,
optionally after torch.cuda.init() (argv[1] = 'init') or with extra work first."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2604_14650_b200 as lpm
from paper_2604_14650_b200 import store as st
from paper_2604_14650_b200.fib import Prefix

if len(sys.argv) > 1 and sys.argv[1] == "init":
    torch.cuda.init()
fib = lpm.workload_fib(1)
t0 = time.perf_counter()
store = st.FibStore(fib, 0, value_bytes=1)
create_ms = (time.perf_counter() - t0) * 1e3
rng = np.random.default_rng(1)
rules = fib.rules
times, builds = [], []
for _ in range(5):
    idx = rng.integers(0, len(rules), 1000)
    store.stage([st.UpdateOp(st.ANNOUNCE, Prefix(int(rules[i]["value_hi"]) << 64, int(rules[i]["length"]),
                                                 int(rng.integers(1, 255)))) for i in idx])
    t0 = time.perf_counter()
    store.commit()
    times.append(round((time.perf_counter() - t0) * 1e3, 2))
    builds.append(round(store.stats.last_build_ms, 2))
store.close()
print(json.dumps({"argv": sys.argv[1:], "create_ms": round(create_ms, 1), "commit_ms": times, "build_ms": builds}))

"""Where does the first FibStore commit's time go? (VERDICT r1 'store cold start')
Times, in one fresh process: the first device build, a FibStore create, and five
commits of 1,000 announces each (wall time and the store's own build time).
    python tools/store_cold.py [C1|C2]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2604_14650_b200 as lpm
from paper_2604_14650_b200.fib import Prefix

wl = sys.argv[1] if len(sys.argv) > 1 else "C1"
info = lpm.workload_info(wl)
fib = lpm.workload_fib(info.fib_kind)
torch.cuda.init()
res = {"workload": wl}
t0 = time.perf_counter()
st = lpm.FibStore(fib, 0, value_bytes=info.value_bytes)
torch.cuda.synchronize()
res["create_ms"] = (time.perf_counter() - t0) * 1e3
res["create_build_ms"] = st.stats.last_build_ms
rng = np.random.default_rng(1)
rules = fib.rules
commits = []
for _ in range(5):
    idx = rng.integers(0, len(rules), 1000)
    ops = [lpm.UpdateOp(3, Prefix(int(rules[i]["value_hi"]) << 64, int(rules[i]["length"]), int(rng.integers(1, 255))))
           for i in idx]
    st.stage(ops)
    t0 = time.perf_counter()
    st.commit()
    commits.append({"commit_ms": (time.perf_counter() - t0) * 1e3, "build_ms": st.stats.last_build_ms})
res["commits"] = commits
st.close()
print(json.dumps(res))

"""Measure the roofline denominators on this GPU: L2 random-gather and smem bandwidth."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_14650_b200 as lpm  # noqa: E402

res = {"smem_gbs": lpm.probe_smem(0), "l2_gather_gbs": {}}
for mb in (1, 3.3, 16, 32, 64, 256):
    for line in (32, 128):
        res["l2_gather_gbs"][f"{mb}MB/{line}B"] = lpm.probe_l2_gather(0, int(mb * (1 << 20)), line)
print(json.dumps(res, indent=1))

"""Shared-memory bank-conflict model of Phase A (host only, no GPU): replays the
kernel's 4-probe searches of the staged levels for a workload's queries in warp
order and counts LDS.64 wavefronts per warp instruction under two models
(whole warp / half-warps: an 8-byte word occupies a bank pair, a wavefront serves
one word per bank pair). Also replays the same queries sorted by the node they
probe at a given level inside each CTA's batch of 1,024 (the CTA-level reorder of
DESIGN §10), to bound what such a reorder could save.
    python tools/bank_sim.py [C1|C2|C3b] [queries]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2604_14650_b200 as lpm

wl = sys.argv[1] if len(sys.argv) > 1 else "C1"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
info = lpm.workload_info(wl)
fib = lpm.workload_fib(info.fib_kind)
tree = lpm.build_tree(lpm.build_intervals(fib), info.value_bytes)
g = tree.geometry
q = lpm.workload_queries_host(wl, fib, 0, nq)
keys = np.minimum(q.view(np.uint64).reshape(-1, 2)[:, 1], np.uint64(0xFFFFFFFFFFFFFFFE))
T = min(g.image_levels, g.depth)
img = tree.lines[g.image_start:]
off = [(g.level_start[l] // 16) * 15 for l in range(T + 1)]  # word offset of level l in the image


def descend(keys):
    """Per level 1..T-1 and probe 0..3: the image word each query reads; node at each level."""
    n = np.zeros(len(keys), np.int64)
    words = {}
    nodes = {0: n.copy()}
    root = tree.lines[:16]
    c = np.zeros(len(keys), np.int64)
    # root (constant bank) then levels 1..T-1 from the image
    for l in range(T):
        c = np.zeros(len(keys), np.int64)
        for step, bit in enumerate((8, 4, 2, 1)):
            pos = c | (bit - 1)
            if l == 0:
                k = root[pos]
            else:
                w = off[l] + n * 15 + pos
                words[(l, step)] = w
                k = img[w]
            c = np.where(k <= keys, c | bit, c)
        n = n * 16 + c
        nodes[l + 1] = n.copy()
    return words, nodes


def wavefronts(w, half):
    """LDS.64 wavefronts per warp instruction for word addresses w (multiple of 32);
    half = lanes served together (32, 16 or 8)."""
    w = w.reshape(-1, half)
    tot = 0
    for row in w:
        u = np.unique(row)
        cnt = np.bincount(u % 16, minlength=16)
        tot += max(1, cnt.max())
    return tot


def report(label, keys):
    words, _ = descend(keys)
    print(label)
    for half in (32, 16, 8):
        per_level = {}
        for (l, step), w in words.items():
            per_level[l] = per_level.get(l, 0) + wavefronts(w[: len(w) // 32 * 32], half)
        nw = len(keys) // 32
        tot = sum(per_level.values())
        print(f"  model {half}-lane groups: {tot / nw / 32:.3f} wavefronts/query "
              f"({tot / nw / (4 * (T - 1)):.2f} per LDS); by level " +
              ", ".join(f"L{l} {v / nw / 32:.3f}" for l, v in sorted(per_level.items())))


report(f"{wl}: {nq} queries, staged levels 0..{T - 1} (root in the constant bank), warp order", keys)
_, nodes = descend(keys)
for lvl in range(2, T):
    order = np.concatenate([b * 1024 + np.argsort(nodes[lvl][b * 1024:(b + 1) * 1024], kind="stable")
                            for b in range(len(keys) // 1024)])
    report(f"sorted inside each 1,024-query batch by the node probed at level {lvl}", keys[order])

"""Host model (no GPU) of the split-plane Phase A (lookup_kernel.cuh PLANES): every staged
level stored as a plane of its nodes' 15 high words followed by a plane of their low
words, probed with one LDS.32 of the high word;
the low word is read only when some lane of the warp ties on the high word (a
warp-uniform branch). Replays a workload's queries in warp order and reports, per
level and probe, the per-lane tie rate, the share of warp steps with any tie (1, 2 and 4
tiles per warp sharing the branch), and LDS.32 wavefronts per warp load under a 32-bank
model, next to the LDS.64 model of tools/bank_sim.py.
    python tools/hilo_sim.py [C1|C2|C3a|C3b] [queries]"""
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
off = [(g.level_start[l] // 16) * 15 for l in range(T + 1)]


def max_load(addr_words, banks, lanes):
    """Wavefronts per warp instruction: distinct words per bank, max over banks, summed over lane groups."""
    w = addr_words.reshape(-1, lanes)
    tot = 0
    for row in w:
        u = np.unique(row)
        tot += max(1, np.bincount(u % banks, minlength=banks).max())
    return tot / (len(addr_words) // 32)


n = np.zeros(len(keys), np.int64)
qhi = keys >> np.uint64(32)
nw = len(keys) // 32
print(f"{wl}: {nq} queries, staged levels 1..{T - 1}")
tot32 = tot64 = tot_slow = 0.0
for l in range(T):
    c = np.zeros(len(keys), np.int64)
    for step, bit in enumerate((8, 4, 2, 1)):
        pos = c | (bit - 1)
        if l == 0:
            k = tree.lines[:16][pos]
        else:
            k = img[off[l] + n * 15 + pos]
            tie = (k >> np.uint64(32)) == qhi
            any1 = tie.reshape(-1, 32).any(axis=1)
            any2 = tie[: nw // 2 * 64].reshape(-1, 64).any(axis=1)
            any4 = tie[: nw // 4 * 128].reshape(-1, 128).any(axis=1)
            nodes_l = (g.level_start[l + 1] - g.level_start[l]) // 16
            hi_word = off[l] * 2 + n * 15 + pos            # 4-byte word index in the level's high plane
            lo_word = hi_word + nodes_l * 15               # the low plane follows the high plane
            w32 = max_load(hi_word, 32, 32)
            w64 = max_load(off[l] + n * 15 + pos, 16, 16) * 1.0
            # slow path: the tying lanes' low-word loads (one more LDS.32, only those lanes)
            slow = 0.0
            rows = np.nonzero(any1)[0]
            for r in rows[:4000]:
                sel = tie[r * 32:(r + 1) * 32]
                u = np.unique(lo_word[r * 32:(r + 1) * 32][sel])
                slow += max(1, np.bincount(u % 32, minlength=32).max())
            slow = slow / max(1, min(len(rows), 4000)) * any1.mean()
            tot32 += w32; tot64 += w64; tot_slow += slow
            print(f"  L{l} probe {step}: tie/lane {tie.mean() * 100:6.3f} %  warp steps with a tie: 1 tile {any1.mean() * 100:5.1f} %"
                  f"  2 tiles {any2.mean() * 100:5.1f} %  4 tiles {any4.mean() * 100:5.1f} %   LDS.32 {w32:4.2f} wf (+{slow:4.2f} low words)"
                  f"  LDS.64 {w64:4.2f} wf")
        c = np.where(k <= keys, c | bit, c)
    n = n * 16 + c
print(f"  per 32-query tile: LDS.64 model {tot64:.1f} wavefronts, split planes {tot32:.1f} + {tot_slow:.1f} low-word loads")

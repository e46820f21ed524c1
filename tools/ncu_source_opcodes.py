"""Aggregate an ncu source page (ncu -i rep --page source --csv) by SASS opcode:
warp instructions per query and per 32-query tile, L1 tag requests, shared-memory
wavefronts, L2 sectors and the share of stall samples.

usage: python tools/ncu_source_opcodes.py source.csv <queries>"""
import collections
import csv
import sys

KEEP = ("LDG", "STG", "LDS", "TLD", "SHFL", "LDC", "STS")


def main(path, queries):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        toks = [t for t in r[ix["Source"]].split() if not t.startswith("@")]
        if not toks:
            continue
        op = toks[0] if toks[0].startswith(KEEP) else toks[0].split(".")[0]
        a = agg[op]
        for slot, col in enumerate(("Instructions Executed", "L1 Tag Requests Global", "L1 Wavefronts Shared",
                                    "# Samples", "L2 Theoretical Sectors Global")):
            a[slot] += int(r[ix[col]] or 0)
    tot = sum(a[0] for a in agg.values())
    samples = sum(a[3] for a in agg.values())
    print(rows[0][1])
    print(f"warp instructions per query {tot / queries:.3f} (per 32-query tile {32 * tot / queries:.1f})")
    print(f"{'opcode':24s} {'inst/query':>10s} {'inst/tile':>10s} {'L1 tag req/q':>13s} {'smem wavefronts/q':>18s} "
          f"{'L2 sectors/q':>13s} {'stall samples':>14s}")
    for op, a in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if a[0] == 0:
            continue
        print(f"{op:24s} {a[0] / queries:10.4f} {32 * a[0] / queries:10.2f} {a[1] / queries:13.4f} "
              f"{a[2] / queries:18.4f} {a[4] / queries:13.3f} {100 * a[3] / samples:13.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))

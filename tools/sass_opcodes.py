"""Opcode census of the bench kernels' SASS (cuobjdump, no GPU needed) plus their
ptxas register/spill lines: the evidence that the lookup uses the TMA bulk copy
(UBLKCP) on an mbarrier (SYNCS.*), 256-bit L2 line loads (LDG.E.ELL2.256), texture
line fetches (TLD), shuffles (SHFL) and no local-memory spills.
    python tools/sass_opcodes.py > profiles/r02_sass_opcodes.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OBJ = ROOT / "build" / "obj"
# (label, object, template args of lpm6_lookup_kernel<DEPTH, VB, TILES, THREADS, MINB, CHECKED, INPUT, LEAFS, TEXL,
#  LEAFTEX, HALF, TAS, PBSEQ>)
KERNELS = [
    ("C2/C4 bench kernel: line path 1, half-line leaves, 4 tiles per warp, PBSEQ (depth 5, u16)", "lookup_vb2.cu.o",
     "ILi5ELi2ELi4ELi1024ELi1ELb0ELi0ELb0ELi1ELi1ELb1ELi4ELb1ELi0EE"),
    ("C2/C4 one tile per warp, line path 1, half-line leaves", "lookup_vb2.cu.o",
     "ILi5ELi2ELi1ELi1024ELi1ELb0ELi0ELb0ELi1ELi1ELb1ELi4ELb0ELi0EE"),
    ("C1/C3b packed kernel: line path 1, 2 tiles per warp, PBSEQ (depth 4, u8)", "lookup_vb1.cu.o",
     "ILi4ELi1ELi2ELi1024ELi1ELb0ELi0ELb0ELi0ELi1ELb0ELi4ELb1ELi0EE"),
    ("C1 bench kernel (v20): line path 1, 2 tiles per warp, split planes on levels 1-2 (PLANES = 3)", "lookup_vb1.cu.o",
     "ILi4ELi1ELi2ELi1024ELi1ELb0ELi0ELb0ELi0ELi1ELb0ELi4ELb1ELi3EE"),
    ("C3b bench kernel (v20): line path 4, 2 tiles per warp, split planes on every staged level", "lookup_vb1.cu.o",
     "ILi4ELi1ELi2ELi1024ELi1ELb0ELi0ELb0ELi0ELi3ELb0ELi4ELb1ELi8EE"),
    ("C3a bench kernel: line path 4, 2 tiles per warp, PBSEQ", "lookup_vb1.cu.o",
     "ILi4ELi1ELi2ELi1024ELi1ELb0ELi0ELb0ELi0ELi3ELb0ELi4ELb1ELi0EE"),
    ("C1 one tile per warp, line path 1", "lookup_vb1.cu.o", "ILi4ELi1ELi1ELi1024ELi1ELb0ELi0ELb0ELi0ELi1ELb0ELi4ELb0ELi0EE"),
    ("C1 line path 2 (split leaves)", "lookup_vb1.cu.o", "ILi4ELi1ELi1ELi1024ELi1ELb0ELi0ELb0ELi0ELi2ELb0ELi4ELb0ELi0EE"),
    ("C0 leaf image (depth 2, u8)", "lookup_vb1.cu.o", "ILi2ELi1ELi1ELi1024ELi1ELb0ELi0ELb1ELi0ELi0ELb0ELi0ELb0ELi0EE"),
]
WATCH = ["UBLKCP", "SYNCS", "ELECT", "LDS", "LDG", "TLD", "SHFL", "VOTE", "POPC", "PRMT", "ISETP", "STG", "LDL", "STL",
         "BRA", "EXIT"]


def sass(obj, tag):
    names = subprocess.run(["cuobjdump", "-sass", str(OBJ / obj)], capture_output=True, text=True).stdout
    fn = next(m.group(1) for m in re.finditer(r"Function : (\S+)", names) if tag in m.group(1))
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, str(OBJ / obj)], capture_output=True, text=True).stdout
    ops = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops.append(m.group(2))
    return fn, ops


def ptxas(obj, fn):
    log = (OBJ / (obj + ".ptxas.log")).read_text().splitlines()
    for i, line in enumerate(log):
        if fn in line:
            return " | ".join(x.strip().replace("ptxas info    : ", "") for x in log[i + 2:i + 4])
    return "?"


def main():
    for label, obj, tag in KERNELS:
        fn, ops = sass(obj, tag)
        c = collections.Counter(ops)
        full = collections.Counter(o.split(".")[0] for o in ops)
        print(f"== {label}\n   {fn}\n   ptxas: {ptxas(obj, fn)}")
        print(f"   static SASS instructions: {len(ops)}")
        print("   " + ", ".join(f"{k} {full.get(k, 0)}" for k in WATCH))
        wide = sorted((k, v) for k, v in c.items() if any(s in k for s in ("LDG", "TLD", "UBLKCP", "SYNCS", "LDS", "STG")))
        print("   variants: " + ", ".join(f"{k} {v}" for k, v in wide))
        print()


if __name__ == "__main__":
    sys.exit(main())

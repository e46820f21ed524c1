"""Host side of the path: FIB model, interval sweep and B200 tree layout.

Python mirror of the reference's fib-model / interval-engine / lbtree-core
surface (fib.hpp:74-121, intervals.hpp:18-47, tree.hpp:18-88); the work is done
by the C++ in ``csrc/lpm6`` through the C ABI. Names, argument meaning and
error behaviour follow the reference: failures raise :class:`Lpm6Error` whose
``code`` is the reference ``Errc`` name.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import BuildOpts_t, Geometry_t, Lpm6Error, Prefix_t, WorkloadInfo_t, check, lib

# Memory layout of lpm6::Prefix (fib.hpp:22-29) / lpm6cu_prefix.
PREFIX_DTYPE = np.dtype([("value_lo", "<u8"), ("value_hi", "<u8"), ("length", "<i4"),
                         ("next_hop", "<u4"), ("reserved", "<u8")])
assert PREFIX_DTYPE.itemsize == 32

UNRESOLVED = 0xFFFFFFFF          # types.hpp:17
SENTINEL_KEY = 0xFFFFFFFFFFFFFFFF  # types.hpp:21
MAX_QUERY_KEY = SENTINEL_KEY - 1   # types.hpp:25


@dataclass(frozen=True)
class Prefix:
    """One rule: 128-bit value (text order), length 0..64, next hop (fib.hpp:22-29)."""
    value: int
    length: int
    next_hop: int

    def top64(self) -> int:
        return self.value >> 64


def parse_prefix(text: str) -> tuple[Prefix, bool]:
    """``"<ipv6>/<len> <next_hop>"`` -> (Prefix, host_bits_masked) (fib.cpp:72-105)."""
    out = Prefix_t()
    masked = C.c_int(0)
    check(lib().lpm6_parse_prefix(text.encode(), C.byref(out), C.byref(masked)))
    return Prefix((out.value_hi << 64) | out.value_lo, out.length, out.next_hop), bool(masked.value)


class FibTable:
    """Rule set with unique (value, length) pairs and a no-match next hop (fib.hpp:74-105)."""

    def __init__(self, default_next_hop: int = 0, rules: np.ndarray | None = None):
        self.default_next_hop = int(default_next_hop)
        self._rules = np.zeros(0, PREFIX_DTYPE) if rules is None else np.ascontiguousarray(rules, PREFIX_DTYPE)
        self._index: dict[tuple[int, int], int] | None = None

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_prefixes(cls, prefixes, default_next_hop: int = 0) -> "FibTable":
        t = cls(default_next_hop)
        for p in prefixes:
            t.insert(p)
        return t

    def _idx(self) -> dict[tuple[int, int], int]:
        if self._index is None:
            self._index = {(int(r["value_hi"]), int(r["length"])): i for i, r in enumerate(self._rules)}
        return self._index

    def insert(self, p: Prefix) -> None:
        if p.next_hop == UNRESOLVED:
            raise Lpm6Error(4, "next hop 4294967295 is reserved")
        key = (p.value >> 64, p.length)
        if key in self._idx():
            raise Lpm6Error(5, f"duplicate prefix /{p.length}")
        self._append(p, key)

    def insert_or_replace(self, p: Prefix) -> bool:
        if p.next_hop == UNRESOLVED:
            raise Lpm6Error(4, "next hop 4294967295 is reserved")
        key = (p.value >> 64, p.length)
        i = self._idx().get(key)
        if i is None:
            self._append(p, key)
            return False
        self._rules[i]["next_hop"] = p.next_hop
        return True

    def _append(self, p: Prefix, key) -> None:
        row = np.zeros(1, PREFIX_DTYPE)
        row["value_lo"] = p.value & 0xFFFFFFFFFFFFFFFF
        row["value_hi"] = p.value >> 64
        row["length"] = p.length
        row["next_hop"] = p.next_hop
        self._idx()[key] = len(self._rules)
        self._rules = np.concatenate([self._rules, row])

    # -- access ---------------------------------------------------------------
    @property
    def rules(self) -> np.ndarray:
        """Structured array in lpm6::Prefix layout (pass ``rules.ctypes.data`` to the C ABI)."""
        return self._rules

    def __len__(self) -> int:
        return len(self._rules)

    def entries(self) -> list[Prefix]:
        return [Prefix((int(r["value_hi"]) << 64) | int(r["value_lo"]), int(r["length"]), int(r["next_hop"]))
                for r in self._rules]


def load_fib(text: str) -> FibTable:
    """Text FIB (fib.cpp:165-195): '#' comments, last duplicate wins, /65+ skipped."""
    fib = FibTable()
    for line_no, line in enumerate(text.splitlines(), 1):
        s = line.split("#", 1)[0].strip()
        if not s:
            continue
        try:
            p, _ = parse_prefix(s)
        except Lpm6Error as e:
            if e.code == "UnsupportedPrefixLength":
                continue
            raise Lpm6Error(e.status, f"line {line_no}: {e}") from None
        fib.insert_or_replace(p)
    return fib


@dataclass
class IntervalMap:
    """Sorted elementary-interval starts and next hops (intervals.hpp:18-24)."""
    boundaries: np.ndarray  # uint64
    next_hops: np.ndarray   # uint32
    default_next_hop: int

    def __len__(self) -> int:
        return len(self.boundaries)


def _rules_ptr(rules: np.ndarray):
    return rules.ctypes.data if len(rules) else None


def build_intervals(fib: FibTable, merge_adjacent: bool = True) -> IntervalMap:
    """2D->1D transform (intervals.cpp:33-93), computed by csrc/lpm6/intervals.cpp."""
    rules = fib.rules
    cap = 2 * len(rules) + 1
    b = np.empty(cap, np.uint64)
    nh = np.empty(cap, np.uint32)
    m = C.c_uint64(0)
    check(lib().lpm6_build_intervals(_rules_ptr(rules), len(rules), fib.default_next_hop, int(merge_adjacent),
                                     b.ctypes.data, nh.ctypes.data, cap, C.byref(m)))
    return IntervalMap(b[: m.value].copy(), nh[: m.value].copy(), fib.default_next_hop)


@dataclass
class Geometry:
    """B200 tree geometry (lpm6cu_geometry; counterpart of tree.hpp:18-33)."""
    k: int
    b: int
    depth: int
    value_bytes: int
    leaf_keys: int
    image_levels: int
    num_keys: int
    leaf_nodes: int
    total_words: int
    image_start: int
    level_nodes: list[int]
    level_start: list[int]
    default_next_hop: int
    leaf_image: int = 0
    leaf_words: int = 16  # 16: 128-byte leaf lines; 8: half-line leaves (layout.hpp)

    @classmethod
    def from_c(cls, g: Geometry_t) -> "Geometry":
        return cls(g.k, g.b, g.depth, g.value_bytes, g.leaf_keys, g.image_levels, g.num_keys, g.leaf_nodes,
                   g.total_words, g.image_start, list(g.level_nodes), list(g.level_start), g.default_next_hop,
                   g.leaf_image, g.leaf_words or 16)

    def to_c(self) -> Geometry_t:
        g = Geometry_t()
        g.k, g.b, g.depth, g.value_bytes, g.leaf_keys = self.k, self.b, self.depth, self.value_bytes, self.leaf_keys
        g.image_levels, g.image_start = self.image_levels, self.image_start
        g.num_keys, g.leaf_nodes, g.total_words = self.num_keys, self.leaf_nodes, self.total_words
        for i in range(len(self.level_nodes)):
            g.level_nodes[i] = self.level_nodes[i]
            g.level_start[i] = self.level_start[i]
        g.default_next_hop = self.default_next_hop
        g.leaf_image = self.leaf_image
        g.leaf_words = self.leaf_words
        return g

    @property
    def tree_bytes(self) -> int:
        return self.total_words * 8

    def memory_footprint(self) -> dict:
        """Exact bytes of the B200 layout (memory_footprint, tree.hpp:76-88)."""
        from ._lib import Footprint_t
        f = Footprint_t()
        g = self.to_c()
        check(lib().lpm6_memory_footprint(C.byref(g), C.byref(f)))
        return {k: getattr(f, k) for k, _ in Footprint_t._fields_}


def ref_memory_footprint(m: int, k: int = 8) -> dict:
    """memory_footprint of the reference's layout for m intervals."""
    from ._lib import Footprint_t
    f = Footprint_t()
    check(lib().lpm6_ref_memory_footprint(m, k, C.byref(f)))
    return {name: getattr(f, name) for name, _ in Footprint_t._fields_}


LEAF_AUTO, LEAF_FULL, LEAF_HALF = 0, 1, 2  # lpm6cu_build_opts.leaf_format


def plan_layout(m: int, value_bytes: int = 1, leaf_format: int = LEAF_AUTO) -> Geometry:
    g = Geometry_t()
    check(lib().lpm6_plan_layout_ex(m, value_bytes, leaf_format, C.byref(g)))
    return Geometry.from_c(g)


@dataclass
class Tree:
    """Host copy of the B200 layout: 128-byte lines (internal: 16 separators; leaf:
    leaf_keys keys + their next hops) and the next hop of every leaf slot."""
    geometry: Geometry
    lines: np.ndarray        # uint64[total_words]
    leaf_values: np.ndarray  # uint32[leaf_nodes * leaf_keys]

    def leaf_keys_array(self) -> np.ndarray:
        """The leaf boundary keys in slot order (sentinels past m)."""
        g = self.geometry
        start = g.level_start[g.depth]
        leaves = self.lines[start: start + g.leaf_nodes * g.leaf_words].reshape(-1, g.leaf_words)
        return leaves[:, : g.leaf_keys].reshape(-1)


def build_tree(imap: IntervalMap, value_bytes: int = 0, leaf_format: int = LEAF_AUTO) -> Tree:
    """Lay out the linearized tree for B200 (csrc/lpm6/layout.cpp; contract S:215-223);
    leaf_format: LEAF_AUTO, LEAF_FULL (128-byte leaf lines) or LEAF_HALF (half-line
    leaves, 2-byte next hops)."""
    g = Geometry_t()
    b = np.ascontiguousarray(imap.boundaries, np.uint64)
    nh = np.ascontiguousarray(imap.next_hops, np.uint32)
    check(lib().lpm6_build_tree_ex(b.ctypes.data, nh.ctypes.data, len(b), imap.default_next_hop, value_bytes,
                                   leaf_format, C.byref(g), None, None))
    lines = np.empty(g.total_words, np.uint64)
    vals = np.empty(g.leaf_nodes * g.leaf_keys, np.uint32)
    check(lib().lpm6_build_tree_ex(b.ctypes.data, nh.ctypes.data, len(b), imap.default_next_hop, value_bytes,
                                   leaf_format, C.byref(g), lines.ctypes.data, vals.ctypes.data))
    return Tree(Geometry.from_c(g), lines, vals)


# ---- reference file formats: PBT1 snapshots, PBTR traces (csrc/lpm6/snapshot.cpp) --

def encode_snapshot(imap: IntervalMap, k: int = 8) -> bytes:
    """PBT1 bytes of ``imap`` in the reference's layout (tree.hpp:90-96)."""
    b = np.ascontiguousarray(imap.boundaries, np.uint64)
    nh = np.ascontiguousarray(imap.next_hops, np.uint32)
    size = C.c_uint64(0)
    check(lib().lpm6_snapshot_encode(b.ctypes.data, nh.ctypes.data, len(b), k, None, 0, C.byref(size)))
    buf = np.empty(size.value, np.uint8)
    check(lib().lpm6_snapshot_encode(b.ctypes.data, nh.ctypes.data, len(b), k, buf.ctypes.data, size.value,
                                     C.byref(size)))
    return buf.tobytes()


def save_snapshot(imap: IntervalMap, path: str, k: int = 8) -> None:
    b = np.ascontiguousarray(imap.boundaries, np.uint64)
    nh = np.ascontiguousarray(imap.next_hops, np.uint32)
    check(lib().lpm6_snapshot_save(b.ctypes.data, nh.ctypes.data, len(b), k, str(path).encode()))


def decode_snapshot(data: bytes, default_next_hop: int = 0) -> tuple[IntervalMap, int]:
    """Validate a PBT1 image; returns (its interval map, k)."""
    raw = np.frombuffer(data, np.uint8)
    m, k = C.c_uint64(0), C.c_uint32(0)
    ptr = raw.ctypes.data if len(raw) else None
    check(lib().lpm6_snapshot_decode(ptr, len(raw), None, None, 0, C.byref(m), C.byref(k)))
    b = np.empty(m.value, np.uint64)
    nh = np.empty(m.value, np.uint32)
    check(lib().lpm6_snapshot_decode(ptr, len(raw), b.ctypes.data, nh.ctypes.data, m.value, C.byref(m),
                                     C.byref(k)))
    return IntervalMap(b, nh, default_next_hop), k.value


def save_trace(keys: np.ndarray, path: str) -> None:
    """PBTR key trace."""
    k = np.ascontiguousarray(keys, np.uint64)
    check(lib().lpm6_trace_save(k.ctypes.data if len(k) else None, len(k), str(path).encode()))


def trace_count(data: bytes) -> int:
    raw = np.frombuffer(data, np.uint8)
    n = C.c_uint64(0)
    check(lib().lpm6_trace_count(raw.ctypes.data if len(raw) else None, len(raw), C.byref(n)))
    return n.value


# ---- synthetic workloads (BASELINE.json configs) ---------------------------------

WORKLOADS = {"C0": 0, "C1": 1, "C2": 2, "C3a": 3, "C3b": 4, "C4": 5}


@dataclass
class WorkloadInfo:
    id: int
    name: str
    fib_kind: int
    n_queries: int
    chunk: int
    value_bytes: int


def workload_info(workload: int | str) -> WorkloadInfo:
    wid = WORKLOADS[workload] if isinstance(workload, str) else int(workload)
    i = WorkloadInfo_t()
    check(lib().lpm6_workload_info_get(wid, C.byref(i)))
    return WorkloadInfo(i.id, i.name.decode(), i.fib_kind, i.n_queries, i.chunk, i.value_bytes)


_fib_cache: dict[int, FibTable] = {}


def workload_fib(fib_kind: int) -> FibTable:
    """The seeded synthetic FIB of a workload family (csrc/lpm6/workload.cpp)."""
    if fib_kind not in _fib_cache:
        n = C.c_uint64(0)
        dflt = C.c_uint32(0)
        check(lib().lpm6_workload_fib(fib_kind, None, 0, C.byref(n), C.byref(dflt)))
        rules = np.zeros(n.value, PREFIX_DTYPE)
        check(lib().lpm6_workload_fib(fib_kind, rules.ctypes.data, n.value, C.byref(n), C.byref(dflt)))
        _fib_cache[fib_kind] = FibTable(dflt.value, rules)
    return _fib_cache[fib_kind]


def workload_queries_host(workload: int | str, fib: FibTable, first: int, n: int, threads: int = 8) -> np.ndarray:
    """Addresses [first, first+n) as uint64[n, 2] (lo, hi), generated on the host."""
    wid = WORKLOADS[workload] if isinstance(workload, str) else int(workload)
    out = np.empty((n, 2), np.uint64)
    rules = fib.rules
    check(lib().lpm6_workload_queries_host(wid, _rules_ptr(rules), len(rules), first, n, out.ctypes.data,
                                           threads))
    return out


def build_opts(merge_adjacent: bool = True, value_bytes: int = 0, leaf_format: int = LEAF_AUTO) -> BuildOpts_t:
    o = BuildOpts_t()
    o.leaf_format = leaf_format
    o.merge_adjacent = int(merge_adjacent)
    o.value_bytes = value_bytes
    return o

"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

* ``Oracle``    : oracle/liblpm6oracle.so, our plain-C restatement of the
                  reference algorithm (lpm6_oracle.c, each function cites the
                  reference file:line it follows).
* ``RefOracle`` : oracle/_ref/liblpm6ref.so, the reference's own fib.cpp +
                  intervals.cpp compiled in place (oracle/Makefile `ref`).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liblpm6oracle.so"
REF_SO = HERE / "_ref" / "liblpm6ref.so"

P = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int


class Geometry(C.Structure):
    _fields_ = [("k", C.c_int32), ("b", C.c_int32), ("depth", C.c_int32), ("pad", C.c_int32),
                ("num_keys", U64), ("allocated_leaf_nodes", U64), ("leaf_start", U64),
                ("level_start", U64 * 16)]


class Index(C.Structure):
    _fields_ = [("boundaries", P), ("next_hops", P), ("m", U64), ("keys", P), ("values", P),
                ("g", C.POINTER(Geometry))]


def build(force: bool = False) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    if Path(os.environ.get("LPM6_REF_DIR", "/root/reference/proj")).exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class Oracle:
    """The C restatement."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO))
        L.orc_build_intervals.argtypes = [P, U64, U32, I32, P, P, C.POINTER(U64)]
        L.orc_build_intervals.restype = I32
        L.orc_lookup_interval.argtypes = [P, P, U64, U64]
        L.orc_lookup_interval.restype = U32
        L.orc_lookup_linear.argtypes = [P, U64, U32, U64, U64]
        L.orc_lookup_linear.restype = U32
        L.orc_plan_geometry.argtypes = [U64, I32, C.POINTER(Geometry)]
        L.orc_plan_geometry.restype = None
        L.orc_child_key_start.argtypes = [C.POINTER(Geometry), I32, U64, I32]
        L.orc_child_key_start.restype = U64
        L.orc_total_key_slots.argtypes = [C.POINTER(Geometry)]
        L.orc_total_key_slots.restype = U64
        L.orc_build_tree.argtypes = [P, P, U64, I32, C.POINTER(Geometry), P, P]
        L.orc_build_tree.restype = None
        L.orc_search_scalar.argtypes = [P, C.POINTER(Geometry), U64]
        L.orc_search_scalar.restype = U64
        L.orc_search_branchfree.argtypes = [P, C.POINTER(Geometry), U64]
        L.orc_search_branchfree.restype = U64
        L.orc_lookup_batch.argtypes = [I32, C.POINTER(Index), P, U64, P, I32]
        L.orc_lookup_batch.restype = I32
        L.orc_have_avx512.argtypes = []
        L.orc_have_avx512.restype = I32
        self.L = L

    # interval engine --------------------------------------------------------
    def build_intervals(self, rules: np.ndarray, default_nh: int, merge: bool = True):
        """-> (status, boundaries u64[], next_hops u32[]) (intervals.cpp:33-93)."""
        n = len(rules)
        b = np.empty(2 * n + 1, np.uint64)
        nh = np.empty(2 * n + 1, np.uint32)
        m = U64(0)
        st = self.L.orc_build_intervals(rules.ctypes.data if n else None, n, default_nh, int(merge),
                                        b.ctypes.data, nh.ctypes.data, C.byref(m))
        return st, b[: m.value].copy(), nh[: m.value].copy()

    def lookup_interval(self, b: np.ndarray, nh: np.ndarray, key: int) -> int:
        return self.L.orc_lookup_interval(b.ctypes.data, nh.ctypes.data, len(b), key)

    def lookup_linear(self, rules: np.ndarray, default_nh: int, addr: int) -> int:
        return self.L.orc_lookup_linear(rules.ctypes.data if len(rules) else None, len(rules), default_nh,
                                        addr >> 64, addr & 0xFFFFFFFFFFFFFFFF)

    # reference-layout tree ---------------------------------------------------
    def plan_geometry(self, m: int, k: int = 8) -> Geometry:
        g = Geometry()
        self.L.orc_plan_geometry(m, k, C.byref(g))
        return g

    def child_key_start(self, g: Geometry, level: int, node: int, child: int) -> int:
        return self.L.orc_child_key_start(C.byref(g), level, node, child)

    def build_tree(self, b: np.ndarray, nh: np.ndarray, k: int = 8):
        g = self.plan_geometry(len(b), k)
        # KeyArray is 64-byte aligned (tree.hpp:42-74): one node = one cache line.
        slots = self.L.orc_total_key_slots(C.byref(g)) + 16  # +16: SIMD over-read slack
        raw = np.empty(slots + 8, np.uint64)
        off = (-raw.ctypes.data // 8) % 8
        keys = raw[off: off + slots]
        assert keys.ctypes.data % 64 == 0
        keys[:] = 0xFFFFFFFFFFFFFFFF
        values = np.empty(g.allocated_leaf_nodes * k, np.uint32)
        self.L.orc_build_tree(b.ctypes.data, nh.ctypes.data, len(b), k, C.byref(g), keys.ctypes.data,
                              values.ctypes.data)
        return g, keys, values

    def search_scalar(self, keys, g, key: int) -> int:
        return self.L.orc_search_scalar(keys.ctypes.data, C.byref(g), key)

    def search_branchfree(self, keys, g, key: int) -> int:
        return self.L.orc_search_branchfree(keys.ctypes.data, C.byref(g), key)

    def have_avx512(self) -> bool:
        return bool(self.L.orc_have_avx512())

    def lookup_batch(self, variant: int, b, nh, addrs: np.ndarray, threads: int = 1, tree=None):
        """Threaded lookups of uint64[n, 2] (lo, hi) addresses -> (u32[n], variant actually run).

        variant 0: interval oracle; 1: branch-free tree search; 2: restated PlanB
        AVX-512 Listing 1 + B=16 batching (k=8 tree)."""
        if tree is None and variant != 0:
            tree = self.build_tree(b, nh, 8)
        ix = Index()
        ix.boundaries = b.ctypes.data
        ix.next_hops = nh.ctypes.data
        ix.m = len(b)
        if tree is not None:
            g, keys, values = tree
            ix.keys = keys.ctypes.data
            ix.values = values.ctypes.data
            ix.g = C.pointer(g)
        else:
            ix.g = C.pointer(self.plan_geometry(len(b), 8))
        n = len(addrs)
        out = np.empty(n, np.uint32)
        a = np.ascontiguousarray(addrs, np.uint64)
        ran = self.L.orc_lookup_batch(variant, C.byref(ix), a.ctypes.data, n, out.ctypes.data, threads)
        return out, ran


class RefOracle:
    """The reference's own code (oracle/_ref/liblpm6ref.so)."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_intervals.argtypes = [P, U64, U32, I32, C.POINTER(P)]
        L.ref_build_intervals.restype = I32
        L.ref_map_size.argtypes = [P]
        L.ref_map_size.restype = U64
        L.ref_map_copy.argtypes = [P, P, P]
        L.ref_map_copy.restype = None
        L.ref_map_free.argtypes = [P]
        L.ref_map_free.restype = None
        L.ref_lookup_interval.argtypes = [P, P, U64, P, I32]
        L.ref_lookup_interval.restype = None
        L.ref_lookup_linear.argtypes = [P, U64, U32, P, U64, P]
        L.ref_lookup_linear.restype = I32
        L.ref_linear_keys.argtypes = [P, U64, U32, P, U64, P, I32]
        L.ref_linear_keys.restype = I32
        L.ref_parse_prefix.argtypes = [C.c_char_p, P, C.POINTER(I32)]
        L.ref_parse_prefix.restype = I32
        L.ref_prefix_to_range.argtypes = [P, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]
        L.ref_prefix_to_range.restype = None
        L.ref_synth_fib.argtypes = [U64, U64, P]
        L.ref_synth_fib.restype = I32
        self.L = L

    def error(self) -> str:
        return self.L.ref_last_error().decode()

    def build_intervals(self, rules: np.ndarray, default_nh: int, merge: bool = True):
        """-> (status, handle or None)."""
        h = P()
        st = self.L.ref_build_intervals(rules.ctypes.data if len(rules) else None, len(rules), default_nh,
                                        int(merge), C.byref(h))
        return st, (RefMap(self, h) if st == 0 else None)

    def lookup_linear(self, rules: np.ndarray, default_nh: int, addrs: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(addrs, np.uint64)
        out = np.empty(len(a), np.uint32)
        st = self.L.ref_lookup_linear(rules.ctypes.data if len(rules) else None, len(rules), default_nh,
                                      a.ctypes.data, len(a), out.ctypes.data)
        assert st == 0, self.error()
        return out

    def linear_keys(self, rules: np.ndarray, default_nh: int, keys: np.ndarray, threads: int = 8) -> np.ndarray:
        k = np.ascontiguousarray(keys, np.uint64)
        out = np.empty(len(k), np.uint32)
        st = self.L.ref_linear_keys(rules.ctypes.data if len(rules) else None, len(rules), default_nh,
                                    k.ctypes.data, len(k), out.ctypes.data, threads)
        assert st == 0, self.error()
        return out

    def synth_fib(self, n: int, seed: int, dtype) -> np.ndarray:
        out = np.zeros(n, dtype)
        st = self.L.ref_synth_fib(n, seed, out.ctypes.data)
        assert st == 0, self.error()
        return out


class RefMap:
    def __init__(self, ref: RefOracle, h):
        self.ref = ref
        self.h = h
        m = ref.L.ref_map_size(h)
        self.boundaries = np.empty(m, np.uint64)
        self.next_hops = np.empty(m, np.uint32)
        ref.L.ref_map_copy(h, self.boundaries.ctypes.data, self.next_hops.ctypes.data)

    def lookup(self, keys: np.ndarray, threads: int = 1) -> np.ndarray:
        """lpm6::lookup_interval_oracle per key (intervals.cpp:142-145)."""
        k = np.ascontiguousarray(keys, np.uint64)
        out = np.empty(len(k), np.uint32)
        self.ref.L.ref_lookup_interval(self.h, k.ctypes.data, len(k), out.ctypes.data, threads)
        return out

    def __del__(self):
        try:
            self.ref.L.ref_map_free(self.h)
        except Exception:
            pass

"""BENCH / TEST INFRASTRUCTURE ONLY — ctypes access to oracle/liblpm6work.so, the
synthetic workload generator compiled on its own (oracle/workload_capi.cpp).

bench.py's reference arm uses it to make the seeded FIB and query stream of a
BASELINE config without importing paper_2604_14650_b200, so the process that times
the reference's CPU lookup never maps the product library."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
WORK_SO = HERE / "liblpm6work.so"

NAMES = {"C0": 0, "C1": 1, "C2": 2, "C3a": 3, "C3b": 4, "C4": 5}
PREFIX_DTYPE = np.dtype([("value_lo", "<u8"), ("value_hi", "<u8"), ("length", "<i4"), ("next_hop", "<u4"),
                         ("reserved", "<u8")])


@dataclass
class Info:
    id: int
    name: str
    fib_kind: int
    n_queries: int
    chunk: int
    value_bytes: int


@dataclass
class Fib:
    rules: np.ndarray
    default_next_hop: int

    def __len__(self):
        return len(self.rules)


class Workloads:
    def __init__(self):
        if not WORK_SO.exists():
            import subprocess
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = C.CDLL(str(WORK_SO))
        L.wl_last_error.restype = C.c_char_p
        L.wl_info.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64), C.c_char_p]
        L.wl_fib.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.wl_queries.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int]
        self.L = L

    def _check(self, st):
        if st != 0:
            raise RuntimeError(self.L.wl_last_error().decode())

    def info(self, workload: str | int) -> Info:
        wid = NAMES[workload] if isinstance(workload, str) else int(workload)
        fk, vb, nq, ch = C.c_int(), C.c_uint32(), C.c_uint64(), C.c_uint64()
        name = C.create_string_buffer(8)
        self._check(self.L.wl_info(wid, C.byref(fk), C.byref(vb), C.byref(nq), C.byref(ch), name))
        return Info(wid, name.value.decode(), fk.value, nq.value, ch.value, vb.value)

    def fib(self, fib_kind: int) -> Fib:
        n, d = C.c_uint64(), C.c_uint32()
        self._check(self.L.wl_fib(fib_kind, None, 0, C.byref(n), C.byref(d)))
        rules = np.zeros(n.value, PREFIX_DTYPE)
        self._check(self.L.wl_fib(fib_kind, rules.ctypes.data, n.value, C.byref(n), C.byref(d)))
        return Fib(rules, d.value)

    def queries(self, workload: str | int, fib: Fib, first: int, n: int, threads: int = 8) -> np.ndarray:
        """Addresses [first, first + n) as uint64[n, 2] (lo, hi) — bit-identical to the
        product's workload_queries_host and device QueryGen."""
        wid = NAMES[workload] if isinstance(workload, str) else int(workload)
        out = np.empty((n, 2), np.uint64)
        self._check(self.L.wl_queries(wid, fib.rules.ctypes.data if len(fib.rules) else None, len(fib.rules), first,
                                      n, out.ctypes.data, threads))
        return out

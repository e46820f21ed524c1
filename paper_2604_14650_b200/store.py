"""Rebuild-and-swap FIB store on the GPU (SPEC update-engine).

Python mirror of the reference's FibStore surface: ``stage`` / ``commit`` /
``acquire`` / ``release`` with the same semantics and errors. Each
commit rebuilds the whole FIB on the GPU (csrc/build.cu) on the store's own
stream and publishes it with one pointer swap (csrc/store.cpp); readers pin a
snapshot and never wait on a rebuild. ``release(stream)`` is stream-ordered: the
snapshot's device memory outlives every lookup queued on that stream before the
release.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import Lpm6Error, StoreStats_t, UpdateOp_t, check, lib
from .fib import PREFIX_DTYPE, FibTable, Prefix, _rules_ptr, build_opts

INSERT, DELETE, MODIFY, ANNOUNCE = 0, 1, 2, 3  # lpm6_update_op.kind (include/lpm6cu.h)
KIND_NAMES = {INSERT: "Insert", DELETE: "Delete", MODIFY: "Modify", ANNOUNCE: "Announce"}

# lpm6_update_op / lpm6::UpdateOp: 48 bytes.
UPDATE_DTYPE = np.dtype([("kind", "<u4"), ("reserved0", "<u4"), ("reserved1", "<u8"), ("value_lo", "<u8"),
                         ("value_hi", "<u8"), ("length", "<i4"), ("next_hop", "<u4"), ("reserved", "<u8")])
assert UPDATE_DTYPE.itemsize == 48


@dataclass(frozen=True)
class UpdateOp:
    """One route change; ``next_hop`` of ``prefix`` is ignored for Delete."""
    kind: int
    prefix: Prefix


def parse_update(line: str) -> UpdateOp:
    """``A <ipv6>/<len> <next_hop>`` (announce = insert-or-modify) or
    ``W <ipv6>/<len> [next_hop]`` (withdraw = delete)."""
    op = UpdateOp_t()
    check(lib().lpm6_parse_update(line.encode(), C.byref(op)))
    p = op.prefix
    return UpdateOp(op.kind, Prefix((p.value_hi << 64) | p.value_lo, p.length, p.next_hop))


def load_update_trace(text: str) -> tuple[list[UpdateOp], int]:
    """Parse an update trace; returns (ops, lines that failed to parse)."""
    ops, errors = [], 0
    for line in text.splitlines():
        s = line.split("#", 1)[0].strip()
        if not s:
            continue
        try:
            ops.append(parse_update(s))
        except Lpm6Error:
            errors += 1
    return ops, errors


def ops_array(ops) -> np.ndarray:
    """UpdateOps (or an UPDATE_DTYPE array) as the C ABI's lpm6_update_op array."""
    if isinstance(ops, np.ndarray):
        return np.ascontiguousarray(ops, UPDATE_DTYPE)
    a = np.zeros(len(ops), UPDATE_DTYPE)
    for i, op in enumerate(ops):
        a[i]["kind"] = op.kind
        a[i]["value_lo"] = op.prefix.value & 0xFFFFFFFFFFFFFFFF
        a[i]["value_hi"] = op.prefix.value >> 64
        a[i]["length"] = op.prefix.length
        a[i]["next_hop"] = op.prefix.next_hop
    return a


def _status_list(st: np.ndarray) -> list[str | None]:
    from ._lib import ERRC_NAMES
    return [None if s == 0 else ERRC_NAMES[s - 1] for s in st.tolist()]


def apply_updates(fib: FibTable, ops) -> tuple[FibTable, int, list[str | None]]:
    """The store's staging rule on the host (no GPU): ops applied in order, invalid
    ones skipped. Returns (new FibTable, staged count, per-op error code or None)."""
    a = ops_array(ops)
    rules = fib.rules
    n_out, staged = C.c_uint64(0), C.c_uint64(0)
    st = np.zeros(len(a), np.int32)
    cap = len(rules) + len(a)
    out = np.zeros(max(cap, 1), PREFIX_DTYPE)
    check(lib().lpm6_apply_updates(_rules_ptr(rules), len(rules), a.ctypes.data if len(a) else None, len(a),
                                   out.ctypes.data, cap, C.byref(n_out), C.byref(staged), st.ctypes.data))
    return FibTable(fib.default_next_hop, out[: n_out.value].copy()), staged.value, _status_list(st)


class Snapshot:
    """A pinned (epoch, FIB) pair; use as a context manager or call ``release``."""

    def __init__(self, store: "FibStore", handle: C.c_void_p):
        from .gpu import Fib
        self._store = store
        self._h = handle
        epoch, fib, n = C.c_uint64(0), C.c_void_p(), C.c_uint64(0)
        check(lib().lpm6cu_snapshot_info(handle, C.byref(epoch), C.byref(fib), C.byref(n)))
        self.epoch = epoch.value
        self.num_rules = n.value
        self.fib = Fib(fib.value, store.device, owned=False)

    def rules(self) -> np.ndarray:
        out = np.zeros(max(self.num_rules, 1), PREFIX_DTYPE)
        check(lib().lpm6cu_snapshot_rules(self._h, out.ctypes.data, self.num_rules))
        return out[: self.num_rules]

    def lookup_batch(self, addrs, out=None, stream=None):
        return self.fib.lookup_batch(addrs, out, stream)

    def release(self, stream=None) -> None:
        """Unpin; lookups queued on ``stream`` (default: torch's current stream) before
        this call keep the snapshot's device memory alive until they finish."""
        if self._h is None:
            return
        from .gpu import _stream_handle
        s = _stream_handle(stream)
        self.fib.close()
        h, self._h = self._h, None
        check(lib().lpm6cu_store_release(h, s))

    def __enter__(self) -> "Snapshot":
        return self

    def __exit__(self, *exc) -> None:
        self.release()


@dataclass
class StoreStats:
    epoch: int
    pending_ops: int
    active_rules: int
    retired: int
    reclaimed: int
    commits: int
    last_build_ms: float
    last_publish_us: float
    fences: int = 0


class FibStore:
    """Device-resident rebuild-and-swap FIB store (lpm6cu_store)."""

    def __init__(self, fib: FibTable, device: int = 0, merge_adjacent: bool = True, value_bytes: int = 0):
        h = C.c_void_p()
        opts = build_opts(merge_adjacent, value_bytes)
        rules = fib.rules
        check(lib().lpm6cu_store_create(device, _rules_ptr(rules), len(rules), fib.default_next_hop,
                                        C.byref(opts), C.byref(h)))
        self._h = h
        self.device = device
        self.default_next_hop = fib.default_next_hop

    def stage(self, ops) -> tuple[int, list[str | None]]:
        """Validate and append ops; returns (staged, per-op error code or None)."""
        a = ops_array(ops)
        staged = C.c_uint64(0)
        st = np.zeros(len(a), np.int32)
        check(lib().lpm6cu_store_stage(self._h, a.ctypes.data if len(a) else None, len(a), C.byref(staged),
                                       st.ctypes.data))
        return staged.value, _status_list(st)

    def commit(self) -> int:
        """Rebuild from the staged view on the GPU and publish; returns the active epoch."""
        e = C.c_uint64(0)
        check(lib().lpm6cu_store_commit(self._h, C.byref(e)))
        return e.value

    def acquire(self) -> Snapshot:
        s = C.c_void_p()
        check(lib().lpm6cu_store_acquire(self._h, C.byref(s)))
        return Snapshot(self, s)

    def lookup_batch(self, addrs, out=None, stream=None):
        """acquire -> lookup -> release(stream) on the current snapshot; returns (out, epoch)."""
        with self.acquire() as snap:
            out = snap.lookup_batch(addrs, out, stream)
            if stream is not None:
                snap.release(stream)
            return out, snap.epoch

    def reclaim(self) -> None:
        check(lib().lpm6cu_store_reclaim(self._h))

    @property
    def stats(self) -> StoreStats:
        s = StoreStats_t()
        check(lib().lpm6cu_store_stats_get(self._h, C.byref(s)))
        return StoreStats(s.epoch, s.pending_ops, s.active_rules, s.retired, s.reclaimed, s.commits,
                          s.last_build_ms, s.last_publish_us, s.fences)

    @property
    def epoch(self) -> int:
        return self.stats.epoch

    def close(self) -> None:
        if self._h and self._h.value:
            check(lib().lpm6cu_store_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Device side: the B200 FIB handle and ``lookup_batch`` (include/lpm6cu.h).

``Fib.build(fib).lookup_batch(addrs, out)`` is the drop-in for the reference's
FibTable -> build_intervals -> build_tree -> search_batch/lookup path
(fib.hpp:74-105, intervals.hpp:34, tree.hpp:74). Lookups run only in
the sm_100a kernels of ``csrc/lookup.cu``; without a CUDA device they fail with
``Lpm6Error(code="CudaError")`` — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Geometry_t, KernelConfig_t, Lpm6Error, check, lib
from .fib import FibTable, Geometry, Tree, _rules_ptr, build_opts

_NP_VDT = {1: np.uint8, 2: np.uint16, 4: np.uint32}


def _torch():
    import torch
    return torch


def _stream_handle(stream) -> int | None:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr_len(buf, item: int) -> tuple[int, int, bool]:
    """(pointer, element count, is_device) of a torch tensor or numpy array of `item`-byte elements."""
    if isinstance(buf, np.ndarray):
        if not buf.flags.c_contiguous:
            raise Lpm6Error(9, "buffer must be contiguous")
        return buf.ctypes.data, buf.nbytes // item, False
    torch = _torch()
    if isinstance(buf, torch.Tensor):
        if not buf.is_contiguous():
            raise Lpm6Error(9, "buffer must be contiguous")
        return buf.data_ptr(), buf.numel() * buf.element_size() // item, buf.is_cuda
    raise TypeError(f"unsupported buffer type {type(buf)}")


class Fib:
    """An immutable FIB resident in one GPU's HBM (lpm6cu_fib)."""

    def __init__(self, handle: int, device: int, keepalive=None, owned: bool = True):
        self._h = C.c_void_p(handle)
        self.device = device
        self._keepalive = keepalive
        self._owned = owned  # False: a store snapshot's FIB, freed by the store
        self._vb = None      # next-hop width, cached (a FIB is immutable)

    # -- construction ---------------------------------------------------------
    @classmethod
    def build(cls, fib: FibTable, device: int = 0, merge_adjacent: bool = True, value_bytes: int = 0,
              leaf_format: int = 0) -> "Fib":
        """Host build (FibTable -> intervals -> layout) into device memory. leaf_format:
        0 auto, 1 full 128-byte leaf lines, 2 half-line leaves (2-byte next hops)."""
        h = C.c_void_p()
        opts = build_opts(merge_adjacent, value_bytes, leaf_format)
        rules = fib.rules
        check(lib().lpm6cu_fib_build(device, _rules_ptr(rules), len(rules), fib.default_next_hop, C.byref(opts),
                                     C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def build_device(cls, fib: FibTable, device: int = 0, merge_adjacent: bool = True, value_bytes: int = 0,
                     stream=None, leaf_format: int = 0) -> "Fib":
        """The same build done on the GPU (csrc/build.cu); bit-identical layout."""
        h = C.c_void_p()
        opts = build_opts(merge_adjacent, value_bytes, leaf_format)
        rules = fib.rules
        s = _stream_handle(stream)
        check(lib().lpm6cu_fib_build_device(device, _rules_ptr(rules), len(rules), fib.default_next_hop,
                                            C.byref(opts), s, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def from_intervals(cls, imap, device: int = 0, value_bytes: int = 0, stream=None, leaf_format: int = 0) -> "Fib":
        """Layout-only device build from an IntervalMap (build_tree(map), tree.hpp:74)."""
        h = C.c_void_p()
        opts = build_opts(True, value_bytes, leaf_format)
        b = np.ascontiguousarray(imap.boundaries, np.uint64)
        nh = np.ascontiguousarray(imap.next_hops, np.uint32)
        check(lib().lpm6cu_fib_build_from_intervals(device, b.ctypes.data, nh.ctypes.data, len(b),
                                                    imap.default_next_hop, C.byref(opts), _stream_handle(stream),
                                                    C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def load_snapshot(cls, path: str, device: int = 0, value_bytes: int = 0, default_next_hop: int = 0,
                      stream=None) -> "Fib":
        """PBT1 snapshot file -> device FIB, no interval sweep (load_snapshot_file, tree.hpp:96)."""
        h = C.c_void_p()
        opts = build_opts(True, value_bytes)
        check(lib().lpm6cu_fib_load_snapshot(device, str(path).encode(), default_next_hop, C.byref(opts),
                                             _stream_handle(stream), C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def from_tree(cls, tree: Tree, device: int = 0) -> "Fib":
        h = C.c_void_p()
        g = tree.geometry.to_c()
        lines = np.ascontiguousarray(tree.lines, np.uint64)
        check(lib().lpm6cu_fib_create(device, C.byref(g), lines.ctypes.data, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def wrap_device(cls, geometry: Geometry, lines, device: int) -> "Fib":
        """Over a device tensor the caller owns (e.g. filled by an NCCL broadcast)."""
        h = C.c_void_p()
        g = geometry.to_c()
        check(lib().lpm6cu_fib_wrap_device(device, C.byref(g), lines.data_ptr(), C.byref(h)))
        return cls(h.value, device, keepalive=lines)

    def replicate(self, devices) -> list["Fib"]:
        """Copies of this FIB on `devices` (devices[0] = this FIB's device) by one
        grouped NCCL broadcast in this process (lpm6cu_fib_replicate)."""
        devs = (C.c_int * len(devices))(*devices)
        outs = (C.c_void_p * len(devices))()
        check(lib().lpm6cu_fib_replicate(self._h, devs, len(devices), outs))
        return [Fib(outs[i], devices[i]) for i in range(len(devices))]

    def close(self) -> None:
        if self._h and self._h.value:
            if self._owned:
                lib().lpm6cu_fib_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- introspection --------------------------------------------------------
    @property
    def value_bytes(self) -> int:
        if self._vb is None:
            self._vb = self.geometry.value_bytes
        return self._vb

    @property
    def geometry(self) -> Geometry:
        g = Geometry_t()
        check(lib().lpm6cu_fib_geometry(self._h, C.byref(g)))
        return Geometry.from_c(g)

    def device_lines(self) -> int:
        p = C.c_void_p()
        check(lib().lpm6cu_fib_device_lines(self._h, C.byref(p)))
        return p.value

    def kernel_config(self) -> dict:
        c = KernelConfig_t()
        check(lib().lpm6cu_fib_kernel_config(self._h, C.byref(c)))
        return {"lanes_per_query": c.lanes_per_query, "smem_levels": c.smem_levels,
                "ctas_per_sm": c.ctas_per_sm, "threads_per_cta": c.threads_per_cta,
                "queries_per_lane": c.queries_per_lane, "min_ctas_per_sm": c.min_ctas_per_sm,
                "line_path": c.line_path, "plane_levels": c.plane_levels}

    def set_kernel_config(self, lanes_per_query: int = 0, smem_levels: int | None = None,
                          ctas_per_sm: int = 0, threads_per_cta: int = 0, queries_per_lane: int = 0,
                          min_ctas_per_sm: int = 0, line_path: int = 0, plane_levels: int = 0) -> dict:
        c = KernelConfig_t()
        c.line_path = line_path
        c.plane_levels = plane_levels
        c.lanes_per_query = lanes_per_query
        c.smem_levels = 0xFF if smem_levels is None else smem_levels
        c.ctas_per_sm = ctas_per_sm
        c.threads_per_cta = threads_per_cta
        c.queries_per_lane = queries_per_lane
        c.min_ctas_per_sm = min_ctas_per_sm
        check(lib().lpm6cu_fib_set_kernel_config(self._h, C.byref(c)))
        return self.kernel_config()

    def tune_line_path(self, addrs, out=None, stream=None, reps: int = 3) -> int:
        """Time the line paths (lpm6cu_kernel_config.line_path 0-4) on a representative
        device batch and keep the fastest in the kernel config; returns its number."""
        vb = self.value_bytes
        aptr, n, adev = _ptr_len(addrs, 16)
        if not adev:
            raise Lpm6Error(9, "tune_line_path takes device buffers")
        if out is None:
            torch = _torch()
            dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[vb]
            out = torch.empty(n, dtype=dt, device=addrs.device)
        optr, nout, odev = _ptr_len(out, vb)
        if not odev:
            raise Lpm6Error(9, "tune_line_path takes device buffers")
        if nout < n:
            raise Lpm6Error(9, f"out holds {nout} next hops, need {n}")
        chosen = C.c_uint32()
        check(lib().lpm6cu_fib_tune_line_path(self._h, aptr, n, optr, _stream_handle(stream), reps,
                                              C.byref(chosen)))
        return int(chosen.value)

    def set_checked(self, on: bool = True) -> None:
        """Bounds-checked kernel: never reads outside the tree, records violations."""
        check(lib().lpm6cu_fib_set_checked(self._h, int(on)))

    def violations(self, reset: bool = True) -> int:
        """OR of violation bits since the last reset (1 smem level, 2 L2 level, 4 leaf rank)."""
        v = C.c_uint32(0)
        check(lib().lpm6cu_fib_violations(self._h, C.byref(v), int(reset)))
        return v.value

    def node_visits(self, reset: bool = True) -> int:
        """Checked mode: tree lines visited since the last reset (depth + 1 per query)."""
        v = C.c_uint64(0)
        check(lib().lpm6cu_fib_node_visits(self._h, C.byref(v), int(reset)))
        return v.value

    # -- lookup ---------------------------------------------------------------
    def lookup_batch(self, addrs, out=None, stream=None):
        """Next hops of n 16-byte little-endian u128 addresses.

        ``addrs``: torch CUDA tensor or numpy array whose bytes are n x 16-byte
        addresses (e.g. uint64[n, 2] as (lo, hi) or uint8[n, 16]). ``out``: a
        buffer of n value-width elements on the same side (allocated when None).
        Device buffers: one asynchronous kernel launch on ``stream`` (default:
        torch's current stream). Host buffers: pipelined copy-in/lookup/copy-out,
        returns when ``out`` is filled.
        """
        vb = self.value_bytes
        aptr, n, adev = _ptr_len(addrs, 16)
        if out is None:
            if adev:
                torch = _torch()
                dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[vb]
                out = torch.empty(n, dtype=dt, device=addrs.device)
            else:
                out = np.empty(n, _NP_VDT[vb])
        optr, nout, odev = _ptr_len(out, vb)
        if nout < n:
            raise Lpm6Error(9, f"out holds {nout} next hops, need {n}")
        if adev != odev:
            raise Lpm6Error(9, "addrs and out must both be device or both be host buffers")
        if adev:  # known device buffers: the launch-only entry point
            check(lib().lpm6cu_lookup_batch_device(self._h, aptr, n, optr, _stream_handle(stream)))
        else:
            check(lib().lpm6cu_lookup_batch(self._h, aptr, n, optr, None))
        return out


    def lookup_keys(self, keys, out=None, stream=None):
        """Next hops of n 8-byte keys (search_batch's input). Device
        buffers: one asynchronous kernel launch on ``stream``; host buffers (numpy):
        the pipelined copy path, returns when ``out`` is filled."""
        vb = self.value_bytes
        kptr, n, kdev = _ptr_len(keys, 8)
        if out is None:
            if kdev:
                torch = _torch()
                dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[vb]
                out = torch.empty(n, dtype=dt, device=keys.device)
            else:
                out = np.empty(n, _NP_VDT[vb])
        optr, nout, odev = _ptr_len(out, vb)
        if nout < n:
            raise Lpm6Error(9, f"out holds {nout} next hops, need {n}")
        if kdev != odev:
            raise Lpm6Error(9, "keys and out must both be device or both be host buffers")
        check(lib().lpm6cu_lookup_keys(self._h, kptr, n, optr, _stream_handle(stream) if kdev else None))
        return out

    def search_batch(self, keys, ordinals=None, next_hops=None, stream=None, with_next_hops: bool = True):
        """search_batch: interval ordinals (int32 tensor; SearchResult::
        interval_ordinal) and, unless with_next_hops is False, next hops of n 8-byte
        keys. Device buffers; one kernel launch on ``stream``."""
        torch = _torch()
        vb = self.value_bytes
        kptr, n, kdev = _ptr_len(keys, 8)
        if ordinals is None:
            ordinals = torch.empty(n, dtype=torch.int32, device=keys.device)
        if next_hops is None and with_next_hops:
            dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[vb]
            next_hops = torch.empty(n, dtype=dt, device=keys.device)
        optr, nout, _ = _ptr_len(ordinals, 4)
        if nout < n:
            raise Lpm6Error(9, f"ordinals holds {nout} entries, need {n}")
        hptr = None
        if next_hops is not None:
            hptr, nh, _ = _ptr_len(next_hops, vb)
            if nh < n:
                raise Lpm6Error(9, f"next_hops holds {nh} entries, need {n}")
        check(lib().lpm6cu_search_batch(self._h, kptr, n, optr, hptr, _stream_handle(stream)))
        return ordinals, next_hops

    def lookup_packets(self, frames, n: int, stride: int, dst_offset: int = 38, out=None, stream=None):
        """Next hops of n frames ``stride`` bytes apart in a device buffer, the IPv6
        destination at ``dst_offset`` (network order; 38 = Ethernet + IPv6)."""
        vb = self.value_bytes
        fptr, nbytes, fdev = _ptr_len(frames, 1)
        if n and (n - 1) * stride + dst_offset + 16 > nbytes:
            raise Lpm6Error(9, "frame buffer too small for n frames")
        if out is None:
            torch = _torch()
            dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[vb]
            out = torch.empty(n, dtype=dt, device=frames.device if fdev else "cuda")
        optr, nout, _ = _ptr_len(out, vb)
        if nout < n:
            raise Lpm6Error(9, f"out holds {nout} next hops, need {n}")
        check(lib().lpm6cu_lookup_packets(self._h, fptr, n, stride, dst_offset, optr, _stream_handle(stream)))
        return out


def load_trace(path: str, device: int = 0, stream=None):
    """PBTR trace file -> torch uint64-as-int64 device tensor of its keys."""
    torch = _torch()
    n = C.c_uint64(0)
    check(lib().lpm6cu_trace_load(device, str(path).encode(), None, 0, C.byref(n), None))
    keys = torch.empty(max(n.value, 1), dtype=torch.int64, device=f"cuda:{device}")
    check(lib().lpm6cu_trace_load(device, str(path).encode(), keys.data_ptr(), n.value, C.byref(n),
                                  _stream_handle(stream)))
    return keys[: n.value]


class QueryGen:
    """Device-side generator of a workload's address stream (bit-identical to the host one)."""

    def __init__(self, workload: int | str, fib: FibTable, device: int = 0):
        from .fib import WORKLOADS
        wid = WORKLOADS[workload] if isinstance(workload, str) else int(workload)
        h = C.c_void_p()
        rules = fib.rules
        check(lib().lpm6cu_querygen_create(device, wid, _rules_ptr(rules), len(rules), C.byref(h)))
        self._h = h
        self.device = device

    def run(self, first: int, n: int, out, stream=None):
        ptr, cap, dev = _ptr_len(out, 16)
        if not dev or cap < n:
            raise Lpm6Error(9, "out must be a device buffer of >= n 16-byte addresses")
        check(lib().lpm6cu_querygen_run(self._h, first, n, ptr, _stream_handle(stream)))
        return out

    def close(self):
        if self._h and self._h.value:
            lib().lpm6cu_querygen_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_intervals_device(fib: FibTable, device: int = 0, merge_adjacent: bool = True):
    """Elementary intervals computed on the GPU (csrc/build.cu), returned as an IntervalMap."""
    from .fib import IntervalMap
    rules = fib.rules
    cap = 2 * len(rules) + 1
    b = np.empty(cap, np.uint64)
    nh = np.empty(cap, np.uint32)
    m = C.c_uint64(0)
    check(lib().lpm6cu_build_intervals_device(device, _rules_ptr(rules), len(rules), fib.default_next_hop,
                                              int(merge_adjacent), b.ctypes.data, nh.ctypes.data, cap, C.byref(m)))
    return IntervalMap(b[: m.value].copy(), nh[: m.value].copy(), fib.default_next_hop)


def device_lines(fib_dev: "Fib") -> np.ndarray:
    """Host copy of a device FIB's line array (for bit-exact layout comparisons)."""
    g = fib_dev.geometry
    out = np.empty(g.total_words, np.uint64)
    check(lib().lpm6cu_fib_copy_lines(fib_dev._h, out.ctypes.data, g.total_words))
    return out


def probe_l2_gather(device: int, buffer_bytes: int, line_bytes: int = 128) -> float:
    v = C.c_double(0)
    check(lib().lpm6cu_probe_l2_gather(device, buffer_bytes, line_bytes, C.byref(v)))
    return v.value


def probe_smem(device: int) -> float:
    v = C.c_double(0)
    check(lib().lpm6cu_probe_smem(device, C.byref(v)))
    return v.value

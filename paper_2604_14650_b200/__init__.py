"""B200-native batched IPv6 longest-prefix-match lookup (PlanB, arxiv 2604.14650).

Host C++ builds the FIB (intervals + 16-key/128-byte-node linearized B+-tree);
hand-written sm_100a kernels answer ``lookup_batch``; NCCL (torch.distributed)
replicates the FIB across GPUs. See DESIGN.md.
"""
from ._lib import Lpm6Error
from .fib import (FibTable, Geometry, IntervalMap, Prefix, Tree, WORKLOADS, build_intervals, build_tree,
                  decode_snapshot, encode_snapshot, load_fib, parse_prefix, plan_layout, ref_memory_footprint,
                  save_snapshot, save_trace,
                  trace_count, workload_fib, workload_info, workload_queries_host)
from .gpu import Fib, QueryGen, load_trace, probe_l2_gather, probe_smem
from .store import FibStore, Snapshot, UpdateOp, apply_updates, load_update_trace, parse_update

__all__ = [
    "Lpm6Error", "FibTable", "Geometry", "IntervalMap", "Prefix", "Tree", "WORKLOADS", "build_intervals",
    "build_tree", "load_fib", "parse_prefix", "plan_layout", "workload_fib", "workload_info",
    "workload_queries_host", "Fib", "QueryGen", "probe_l2_gather", "probe_smem", "FibStore", "Snapshot",
    "UpdateOp", "apply_updates", "load_update_trace", "parse_update", "decode_snapshot", "encode_snapshot",
    "save_snapshot", "save_trace", "trace_count", "load_trace", "ref_memory_footprint",
]

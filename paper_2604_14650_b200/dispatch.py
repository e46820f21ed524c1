"""Multi-GPU dispatcher: replicate the FIB, partition query batches, reduce timings.

Lookups shard by query batch with no inter-GPU traffic: rank 0
builds the FIB on the host once, the 128-byte-line tree is broadcast to every
rank with one collective (NCCL over NVLink on GPUs; gloo in the CPU tests), and
each rank resolves its own contiguous slice of the query stream. The only other
collectives are the max-over-ranks reductions of device timings.
"""
from __future__ import annotations

from dataclasses import asdict

import numpy as np

from .fib import FibTable, Geometry, build_intervals, build_tree


def build_on_root(fib: FibTable, rank: int, value_bytes: int = 0):
    """Rank 0: FIB -> intervals -> B200 layout on the host. Other ranks: None."""
    if rank != 0:
        return None
    return build_tree(build_intervals(fib), value_bytes)


def replicate_tree(tree, dist, device, group=None):
    """Broadcast the layout from rank 0: geometry as an object, lines as one tensor.

    Returns (Geometry, lines tensor on `device`). With dist None (one rank) the
    tensor is made from the local tree.
    """
    import torch
    if dist is None:
        return tree.geometry, torch.from_numpy(tree.lines.view(np.int64)).to(device)
    rank = dist.get_rank(group)
    obj = [asdict(tree.geometry) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    geom = Geometry(**obj[0])
    lines = torch.empty(geom.total_words, dtype=torch.int64, device=device)
    if rank == 0:
        lines.copy_(torch.from_numpy(tree.lines.view(np.int64)))
    dist.broadcast(lines, 0, group=group)
    return geom, lines


def broadcast_updates(ops, dist, group=None):
    """Rank 0's batch of route changes on every rank, as the C ABI's op array.

    The rebuild-and-swap store is replicated by replaying: every rank stages the
    same ops and commits, and the device build is deterministic, so all ranks
    publish bit-identical FIBs at the same epoch without moving the tree. One
    broadcast of 48 bytes per op (NCCL on GPUs, gloo in the CPU tests).
    """
    import torch

    from .store import UPDATE_DTYPE, ops_array
    if dist is None:
        return ops_array(ops)
    rank = dist.get_rank(group)
    a = ops_array(ops) if rank == 0 else None
    n = torch.tensor([len(a) if rank == 0 else 0], dtype=torch.int64)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
    if dev is not None:
        n = n.to(dev)
    dist.broadcast(n, 0, group=group)
    count = int(n.item())
    buf = torch.empty(count * UPDATE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    if rank == 0 and count:
        buf.copy_(torch.from_numpy(a.view(np.uint8)))
    if count:
        dist.broadcast(buf, 0, group=group)
    return buf.cpu().numpy().view(UPDATE_DTYPE).copy()


def shard(rank: int, world: int, per_rank: int, total: int | None = None) -> tuple[int, int]:
    """[first, count) of this rank's queries.

    Weak scaling (total None): every rank gets `per_rank` queries, rank r the r-th
    block. Strong scaling: `total` queries split into near-equal contiguous blocks.
    """
    if total is None:
        return rank * per_rank, per_rank
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist, device=None) -> float:
    """Device time of a multi-rank step = the slowest rank's."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def chunk_hash(out) -> int:
    """Position-weighted wrapping int64 sum of a result buffer's 8-byte words (a torch
    uint8 tensor, computed where it lives — on the device for GPU results)."""
    import torch
    words = out.numel() // 8
    weights = (torch.arange(words, dtype=torch.int64, device=out.device) * 0x9E3779B97F4A7C1 + 0x632BE5AB) | 1
    return int((out[: words * 8].view(torch.int64) * weights).sum().item()) & (2**64 - 1)


def combine_digests(mine: dict, dist) -> dict:
    """sha256 over (chunk index, chunk hash) for every chunk of every rank, in chunk
    order: a checksum of checksums that does not depend on how chunks were sharded."""
    import hashlib
    allh = dict(mine)
    if dist is not None:
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, mine)
        for part in parts:
            allh.update(part)
    h = hashlib.sha256()
    for c in sorted(allh):
        h.update(int(c).to_bytes(8, "little") + (allh[c] & (2**64 - 1)).to_bytes(8, "little"))
    return {"sha256": h.hexdigest(), "chunks": len(allh)}

"""World-size-2 tests of the multi-GPU dispatcher's host logic on CPU (gloo).

The GPU path runs the same code with NCCL (bench.py under torchrun): FIB built
once on rank 0, the line array broadcast to every rank, contiguous query
shards, device times reduced with MAX.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import paper_2604_14650_b200 as lpm
    from paper_2604_14650_b200 import dispatch
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        fib = lpm.workload_fib(1)
        tree = dispatch.build_on_root(fib, rank)
        assert (tree is None) == (rank != 0)
        geom, lines = dispatch.replicate_tree(tree, dist, torch.device("cpu"))
        local = lpm.build_tree(lpm.build_intervals(fib))       # what rank 0 built
        ok_lines = bool(np.array_equal(lines.numpy().view(np.uint64), local.lines))
        ok_geom = geom == local.geometry
        per = 1000
        first, count = dispatch.shard(rank, world, per)
        mine = lpm.workload_queries_host("C1", fib, first, count)
        gathered = [torch.zeros(count, 2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine.view(np.int64)))
        full = lpm.workload_queries_host("C1", fib, 0, per * world)
        ok_shards = bool(np.array_equal(torch.cat(gathered).numpy().view(np.uint64), full))
        mx = dispatch.max_over_ranks(float(rank + 1) * 1.5, dist)
        q.put((rank, ok_lines, ok_geom, ok_shards, mx))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))


def test_dispatch_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5, r
        rank, ok_lines, ok_geom, ok_shards, mx = r
        assert ok_lines and ok_geom and ok_shards
        assert mx == 3.0


def _update_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import paper_2604_14650_b200 as lpm
    from paper_2604_14650_b200 import dispatch
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        fib = lpm.workload_fib(0)
        view = fib
        digests = []
        for batch in range(3):
            ops = None
            if rank == 0:  # only rank 0 reads the feed
                text = "\n".join(f"A 2001:db8:{batch}:{i:x}::/64 {1 + i % 200}" for i in range(50))
                text += "\nW 2001:db8:0:1::/64\nW 2001:db8:0:1::/64"  # second withdraw fails on every rank
                ops, _ = lpm.load_update_trace(text)
            arr = dispatch.broadcast_updates(ops, dist)
            view, staged, errs = lpm.apply_updates(view, arr)
            imap = lpm.build_intervals(view)
            digests.append((len(arr), staged, errs.count("UnknownPrefix"), len(imap),
                            int(imap.boundaries.sum(dtype=np.uint64)), int(imap.next_hops.sum())))
        q.put((rank, digests))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e)))


def test_replicated_updates_world2_gloo():
    """Rank 0 parses an update feed and broadcasts the op array; every rank's staging
    (the store's rule) reaches the same FIB, hence the same device build."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_update_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(r[1], list) for r in res), res
    assert res[0][1] == res[1][1]
    for n_ops, staged, unknown, *_ in res[0][1]:
        assert n_ops == 52 and unknown == (1 if staged == 51 else 2)


def test_shard_strong_and_weak():
    from paper_2604_14650_b200 import dispatch
    assert [dispatch.shard(r, 4, 10) for r in range(4)] == [(0, 10), (10, 10), (20, 10), (30, 10)]
    parts = [dispatch.shard(r, 3, 0, total=10) for r in range(3)]
    assert parts == [(0, 4), (4, 3), (7, 3)]
    assert sum(c for _, c in parts) == 10

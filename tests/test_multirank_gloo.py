"""World-size-2 CPU tests (gloo) of the host-side multi-rank logic of the sharded path:
contiguous index sharding, the grid all-reduce decomposition (per-rank partial sums over the
rank's sources add up to the full sum, P:L622-631 is linear in the source weights), the
sharded scalar reductions of Alg. 2 / Eq. (14), max-over-ranks timing and the NCCL-id broadcast
pattern of capi.init_distributed_context (with a stand-in id: NCCL needs a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synthetic import get, make_inputs, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dense
        cfg = get("c1").with_(n=300, m=240)
        x, y, a, b = make_inputs(cfg)
        lam = 30.0
        # --- grid all-reduce decomposition: each rank spreads only its source shard
        lo, hi = shard_range(y.shape[0], rank, world)
        part = dense.direct_sum(x, y[lo:hi], b[lo:hi], lam, 0)
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)
        full = dense.direct_sum(x, y, b, lam, 0)
        err_mv = float(np.abs(t.numpy() - full).max() / np.abs(full).max())
        # --- sharded scalar reductions: sum a log u over the rank's targets, all-reduced
        u = np.exp(np.random.default_rng(0).normal(size=x.shape[0]))
        lo2, hi2 = shard_range(x.shape[0], rank, world)
        s = torch.tensor([float((a[lo2:hi2] * np.log(u[lo2:hi2])).sum())], dtype=torch.float64)
        dist.all_reduce(s)
        err_s = abs(s.item() - float((a * np.log(u)).sum()))
        # --- max-over-ranks timing (bench.py): rank r reports r + 1 ms
        tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        # --- unique-id broadcast pattern (rank 0 creates, everyone receives the same bytes)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, err_mv, err_s, tm.item(), obj[0] == bytes(range(128))))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in [0, 1, 7, 1000, 100_000_001]:
        for world in [1, 2, 3, 8]:
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for (lo, hi), (lo2, _) in zip(ranges, ranges[1:]):
                assert hi == lo2 and hi >= lo
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_decomposition():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err_mv, err_s, tmax, id_ok in res:
        assert err_mv < 1e-15, err_mv
        assert err_s < 1e-14, err_s
        assert tmax == float(world)
        assert id_ok

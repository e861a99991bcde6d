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
        # --- box-restricted grid exchange: global bbox by MIN/MAX all-reduce,
        # every rank spreads its shard, only the touched box is summed across ranks
        from oracle import nfft_ref
        rng2 = np.random.default_rng(11)
        x2, y2 = 0.3 + 0.4 * rng2.random((50, 2)), 0.2 + 0.5 * rng2.random((46, 2))
        w2 = rng2.random(46)
        lo3, hi3 = shard_range(46, rank, world)
        mine = np.concatenate([x2[shard_range(50, rank, world)[0]:shard_range(50, rank, world)[1]], y2[lo3:hi3]])
        mn, mx = torch.from_numpy(mine.min(0)), torch.from_numpy(mine.max(0))
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        centre = 0.5 * (mn.numpy() + mx.numpy())
        rho = (0.5 - 1 / 16) / float(np.sqrt(((mx.numpy() - mn.numpy()) ** 2).sum()))
        n_grid, m_w = 32, 4
        ulo = n_grid * (rho * (mn.numpy() - centre) + 0.5)
        uhi = n_grid * (rho * (mx.numpy() - centre) + 0.5)
        blo = np.maximum(0, np.floor(ulo).astype(int) - m_w)
        bhi = np.minimum(n_grid - 1, np.floor(uhi).astype(int) + m_w + 1)
        sl = tuple(slice(l, h + 1) for l, h in zip(blo, bhi))
        part = nfft_ref.grid_spread(nfft_ref.scale(y2[lo3:hi3], centre, rho), w2[lo3:hi3], n_grid, m_w, 2.0)
        outside = part.copy()
        outside[sl] = 0.0
        box = torch.from_numpy(np.ascontiguousarray(part[sl]))
        dist.all_reduce(box)
        full = nfft_ref.grid_spread(nfft_ref.scale(y2, centre, rho), w2, n_grid, m_w, 2.0)
        rebuilt = np.zeros_like(full)
        rebuilt[sl] = box.numpy()
        err_box = float(np.abs(rebuilt - full).max() / np.abs(full).max()) + float(np.abs(outside).max())
        q.put((rank, err_mv, err_s, tm.item(), obj[0] == bytes(range(128)), err_box, box.numel() < full.size))
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
    for rank, err_mv, err_s, tmax, id_ok, err_box, smaller in res:
        assert err_box < 1e-14 and smaller, err_box
        assert err_mv < 1e-15, err_mv
        assert err_s < 1e-14, err_s
        assert tmax == float(world)
        assert id_ok

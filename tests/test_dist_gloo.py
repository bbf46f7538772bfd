"""Multi-process host logic of the sharded paths on CPU (gloo, world_size 2
and 4): balanced shard ranges, and the row-shard halo exchange -- each rank
exchanges its boundary rows with its neighbours, computes its slab with the
received halos (the C oracle stands in for kernel K3 here, which has its own
GPU parity tests), and the gathered slabs equal the whole-image result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_5245_b200.dist import exchange_halos, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 65536, 1023):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cscan
        from oracle import port as P

        rng = np.random.default_rng(seed)
        img = (rng.random((H, W)) < 0.5).astype(np.uint8)     # every rank builds the same raster
        packed = P.pack_u32(img)
        lo, hi = shard_range(H, rank, world)
        slab = torch.from_numpy(packed[lo:hi].view(np.int32).copy())
        above = torch.empty(slab.shape[1], dtype=torch.int32)
        below = torch.empty(slab.shape[1], dtype=torch.int32)
        works = exchange_halos(slab[0].clone(), slab[-1].clone(), above, below, rank, world)
        for w in works:
            w.wait()
        a = above.numpy().view(np.uint32) if rank > 0 else None
        b = below.numpy().view(np.uint32) if rank < world - 1 else None
        if a is not None:
            assert (a == packed[lo - 1]).all()
        if b is not None:
            assert (b == packed[hi]).all()
        out = cscan.scan_p32_slab(slab.numpy().view(np.uint32), a, b, W, 1)
        gathered = [torch.empty(0) for _ in range(world)] if rank == 0 else None
        obj = [None] * world
        dist.all_gather_object(obj, (lo, hi, out))
        if rank == 0:
            full = np.concatenate([o[2] for o in sorted(obj, key=lambda t: t[0])])
            q.put(bool((full == cscan.scan_p32(packed, W, 1)).all()))
        del gathered
    finally:
        dist.destroy_process_group()


def _worker_rowshard(rank, world, port, H, W, seed, q):
    """RowShardedEdges orchestration (exchange, interior rows while in flight, the two
    boundary rows after) with the C oracle standing in for kernel K3."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cscan
        from oracle import port as P
        from paper_1401_5245_b200.dist import RowShardedEdges

        rng = np.random.default_rng(seed)
        img = (rng.random((H, W)) < 0.5).astype(np.uint8)
        packed = P.pack_u32(img)
        lo, hi = shard_range(H, rank, world)
        slab = torch.from_numpy(packed[lo:hi].view(np.int32).copy())
        calls = []

        def oracle_k3(sl, ab, be, out, r0, r1):
            calls.append((r0, r1, ab is not None, be is not None))
            a = None if ab is None else ab.numpy().view(np.uint32)[: sl.shape[1]]
            b = None if be is None else be.numpy().view(np.uint32)[: sl.shape[1]]
            full = cscan.scan_p32_slab(sl.numpy().view(np.uint32), a, b, W, 1)
            out[r0:r1] = torch.from_numpy(full[r0:r1].view(np.int32))

        def oracle_k3e(sl, ab, be, out):
            n = sl.shape[0]
            calls.append(("ends", ab is not None, be is not None))
            a = None if ab is None else ab.numpy().view(np.uint32)[: sl.shape[1]]
            b = None if be is None else be.numpy().view(np.uint32)[: sl.shape[1]]
            full = cscan.scan_p32_slab(sl.numpy().view(np.uint32), a, b, W, 1)
            out[0] = torch.from_numpy(full[0].view(np.int32))
            out[n - 1] = torch.from_numpy(full[n - 1].view(np.int32))

        rs = RowShardedEdges(slab, W, 1, compute=oracle_k3, compute_ends=oracle_k3e)
        out = rs.step().numpy().view(np.uint32).copy()
        obj = [None] * world
        dist.all_gather_object(obj, (rank, lo, out, calls))
        if rank == 0:
            obj.sort(key=lambda t: t[1])
            full = np.concatenate([o[2] for o in obj])
            ok = bool((full == cscan.scan_p32(packed, W, 1)).all())
            # interior rows [1, n-1) first, without halos; then ONE call for rows
            # 0 and n-1 with the halos that exist at this rank's position
            for r, _, o, c in obj:
                ok &= len(c) == 2 and c[0] == (1, len(o) - 1, False, False) and c[1] == (
                    "ends", r > 0, r < world - 1)
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_edges_orchestration_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker_rowshard, args=(world, _free_port(), 47, 130, 11, q), nprocs=world, join=True)
    assert q.get(timeout=60) is True


@pytest.mark.parametrize("world", [2, 4])
def test_row_shard_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, 61, 200, world, q), nprocs=world, join=True)
    assert q.get(timeout=60) is True

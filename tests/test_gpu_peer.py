"""Peer-memory halos (PeerHaloEdges, bench.py --halo p2p): two or three ranks
on ONE GPU exchange CUDA IPC handles over gloo and each runs a single edge
kernel that reads its neighbour's boundary row straight from the other
process's allocation; on an 8-GPU box the same pointers resolve over NVLink.
The per-step handshake is host-side (stream synchronize + barrier), so no
kernel and no stream waits on another process's memory -- processes that wait
on one another on the device must not share a GPU (B200_PROFILING.md)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cscan
        from oracle import port as P
        from paper_1401_5245_b200.dist import PeerHaloEdges, shard_range

        rng = np.random.default_rng(123)
        img = (rng.random((H, W)) < 0.5).astype(np.uint8)
        packed = P.pack_u32(img)
        lo, hi = shard_range(H, rank, world)
        slab = torch.from_numpy(packed[lo:hi].view(np.int32).copy()).cuda()
        ph = PeerHaloEdges(slab, W, 1)
        out = ph.step().cpu().numpy().view(np.uint32)
        exp = cscan.scan_p32(packed, W, 1)[lo:hi]
        ok = bool((out == exp).all())
        ph.acquire_for_write()              # neighbours done reading before memory goes away
        ph.close()
        res = [None] * world
        dist.all_gather_object(res, ok)
        if rank == 0:
            q.put(all(res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_halo_processes_one_gpu(world, cuda_dev):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _port(), 150, 8192, q), nprocs=world, join=True)
    assert q.get(timeout=120) is True


def _worker_rewrite(rank, world, port, H, W, steps, q):
    """Slabs REWRITTEN every step, with skewed producers: step k's raster is
    fresh random bits; before writing, odd ranks stall their stream on even
    steps and even ranks on odd steps (torch.cuda._sleep), so without the
    handshake a neighbour would read the previous step's boundary rows (or a
    half-written slab)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cscan
        from oracle import port as P
        from paper_1401_5245_b200.dist import PeerHaloEdges, shard_range

        lo, hi = shard_range(H, rank, world)
        rasters = []
        for k in range(steps):
            img = (np.random.default_rng([7, k]).random((H, W)) < 0.5).astype(np.uint8)
            rasters.append(P.pack_u32(img))
        src = torch.from_numpy(np.stack([r[lo:hi] for r in rasters]).view(np.int32)).cuda()
        slab = torch.zeros_like(src[0])
        ph = PeerHaloEdges(slab, W, 1)
        outs = []
        for k in range(steps):
            ph.acquire_for_write()              # neighbours are done with step k-1's rows
            if (k + rank) % 2 == 0:
                torch.cuda._sleep(2_000_000)    # ~1 ms stall before this producer writes
            slab.copy_(src[k])
            outs.append(ph.step().clone())
        torch.cuda.synchronize()
        ok = True
        for k in range(steps):
            exp = cscan.scan_p32(rasters[k], W, 1)[lo:hi]
            ok &= bool((outs[k].cpu().numpy().view(np.uint32) == exp).all())
        ph.acquire_for_write()
        ph.close()
        res = [None] * world
        dist.all_gather_object(res, ok)
        if rank == 0:
            q.put(all(res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_halo_handshake_rewritten_slabs(world, cuda_dev):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker_rewrite, args=(world, _port(), 96, 4096, 12, q), nprocs=world, join=True)
    assert q.get(timeout=180) is True

"""Multi-GPU layer: one process per GPU over torch.distributed (NCCL on the
B200 box, gloo in the CPU tests).  The reference is single-threaded numpy
with no distributed code; this layer is new.

* Batch sharding (configs C2, C5): rank r owns images [lo, hi) of the batch
  (`shard_range`); the images are independent, so there is no collective on
  the data path.
* Row sharding (config C4): rank r owns rows [lo, hi) of one giant raster;
  ranks 0 and G-1 use the border fill on their outer side (bitimage.py:216-223).
  `PeerHaloEdges` (opt-in): the edge kernel reads the neighbours' boundary rows
  straight from their HBM over NVLink (CUDA IPC peer pointers) -- one launch
  per step, ordered by a host-side handshake (stream sync + barrier).
  `RowShardedEdges`: one packed row to each row neighbour by grouped NCCL
  send/recv (8 KiB per message at 65536 px) while the interior rows, which need
  no halo, are computed; the two boundary rows follow the received halos on a
  side stream (one K3e launch), overlapping the interior kernel.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of `total` units for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world, device index).  BITEDGE_SHARE_GPU=1 maps every rank onto
    device 0 -- a functional test of the multi-rank paths on a one-GPU box (the
    timings of such a run mean nothing)."""
    local = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("BITEDGE_SHARE_GPU"):
        local = 0
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), local


def init(backend: str | None = None) -> tuple[int, int]:
    """Initialise the default process group from torchrun's env (no-op at world 1)."""
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = os.environ.get("BITEDGE_DIST_BACKEND") or (
                "nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world


def _needs_host_staging(t: torch.Tensor, group=None) -> bool:
    """gloo has no CUDA send/recv: CUDA rows then travel through host copies
    (the functional multi-rank tests on one GPU; NCCL moves them in HBM)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def exchange_halos(first_row: torch.Tensor, last_row: torch.Tensor, above: torch.Tensor,
                   below: torch.Tensor, rank: int, world: int, group=None):
    """Post the halo exchange of one row slab and return the pending works.

    Sends `first_row` to rank-1 and `last_row` to rank+1; receives rank-1's
    last row into `above` and rank+1's first row into `below`.  At the image
    border (rank 0 above, rank world-1 below) nothing is exchanged and the
    caller passes a NULL halo so the kernel applies the border fill.  Under
    gloo, CUDA rows are staged through host memory and the exchange completes
    before this returns (the returned list is then empty)."""
    if world > 1 and _needs_host_staging(first_row, group):
        h_first, h_last = first_row.cpu(), last_row.cpu()
        h_above, h_below = torch.empty_like(h_first), torch.empty_like(h_last)
        works = exchange_halos(h_first, h_last, h_above, h_below, rank, world, group)
        for w in works:
            w.wait()
        if rank > 0:
            above.copy_(h_above)
        if rank < world - 1:
            below.copy_(h_below)
        return []
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.irecv, above, rank - 1, group))
        ops.append(dist.P2POp(dist.isend, first_row, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.irecv, below, rank + 1, group))
        ops.append(dist.P2POp(dist.isend, last_row, rank + 1, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


class RowShardedEdges:
    """Edges of this rank's row slab of one raster (config C4), with the halo
    exchange overlapped with the interior rows.

    `slab` is an int32 CUDA tensor [rows, S] of MSB-first row words; the
    result lands in `self.out` (same shape)."""

    def __init__(self, slab: torch.Tensor, width: int, border=1, group=None, compute=None,
                 compute_ends=None):
        """`compute(slab, above, below, out, row_lo, row_hi)` computes output rows
        [row_lo, row_hi) of the slab (default: kernel K3 through the C ABI) and
        `compute_ends(slab, above, below, out)` its rows 0 and rows-1 (default:
        K3e, one launch for both); the CPU tests substitute the oracle for both
        to exercise this orchestration."""
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.group = group
        self.slab = slab
        self.width = int(width)
        self.border = border
        self.rows = slab.shape[0]
        s = slab.shape[1]
        # halo buffers padded to a 32-byte multiple so 256-bit loads stay in bounds
        pad = (s + 7) // 8 * 8
        self.above = torch.empty(pad, dtype=slab.dtype, device=slab.device)
        self.below = torch.empty(pad, dtype=slab.dtype, device=slab.device)
        self.out = torch.empty_like(slab)
        if compute is None:
            from . import cuda as _cuda

            def compute(sl, ab, be, out, lo, hi):
                _cuda.edges_halo(sl, ab, be, self.width, self.border, out=out, row_lo=lo,
                                 row_hi=hi)
        if compute_ends is None:
            from . import cuda as _cuda

            def compute_ends(sl, ab, be, out):
                _cuda.edges_halo_ends(sl, ab, be, self.width, self.border, out=out)
        self.compute = compute
        self.compute_ends = compute_ends
        self._side = None

    def step(self) -> torch.Tensor:
        rows, s = self.rows, self.slab.shape[1]
        works = exchange_halos(self.slab[0], self.slab[rows - 1], self.above[:s], self.below[:s],
                               self.rank, self.world, self.group)
        above = self.above if self.rank > 0 else None
        below = self.below if self.rank < self.world - 1 else None
        if self.world == 1:
            self.compute(self.slab, None, None, self.out, 0, rows)
            return self.out
        cuda = self.slab.is_cuda
        if cuda:
            # the two end rows on a side stream behind the exchange, so they
            # overlap the interior kernel instead of following it
            cur = torch.cuda.current_stream(self.slab.device)
            if self._side is None:
                self._side = torch.cuda.Stream(self.slab.device)
            self._side.wait_stream(cur)
            with torch.cuda.stream(self._side):
                for w in works:
                    w.wait()
                self.compute_ends(self.slab, above, below, self.out)   # rows 0 and rows-1
        if rows > 2:  # interior rows need no halo: overlap them with the exchange
            self.compute(self.slab, None, None, self.out, 1, rows - 1)
        if cuda:
            cur.wait_stream(self._side)
        else:
            for w in works:
                w.wait()
            self.compute_ends(self.slab, above, below, self.out)
        return self.out


# CUDA IPC mappings are per allocation and may be opened only once per process:
# several exported buffers can live in one allocation (torch's caching
# allocator), so opened bases are shared and reference-counted here
_IPC_OPEN: dict = {}


def _ipc_open(capi, ct, handle: bytes, off: int) -> int:
    ent = _IPC_OPEN.get(handle)
    if ent is None:
        ptr = ct.c_void_p()
        capi.call("be_ipc_open", ct.create_string_buffer(handle, 64), 0, ct.byref(ptr))
        ent = _IPC_OPEN[handle] = [ptr.value, 0]
    ent[1] += 1
    return ent[0] + off


def _ipc_release(capi, ct, handle: bytes) -> None:
    ent = _IPC_OPEN.get(handle)
    if ent is None:
        return
    ent[1] -= 1
    if ent[1] == 0:
        capi.call("be_ipc_close", ct.c_void_p(ent[0]), 0)
        del _IPC_OPEN[handle]


class PeerHaloEdges:
    """Row-sharded edges whose halo rows are read from the neighbour ranks'
    slabs over NVLink by the edge kernel itself (CUDA IPC peer pointers passed
    as K3's `above` / `below`): no exchange step and one kernel per step -- the
    fused alternative to `RowShardedEdges`' NCCL send/recv (opt-in:
    bench.py --halo p2p).

    Setup exports this rank's slab (`be_ipc_export`), all-gathers the handles
    and opens the row neighbours' (`be_ipc_open`).  Ordering between ranks is a
    host-side handshake on the process group -- no kernel and no stream waits
    on another rank's memory:

        step():               this rank's stream is synchronised (its slab of
                              step s is complete), then a barrier (every
                              neighbour's is), then the edge kernel
        acquire_for_write():  this rank's stream is synchronised (its kernel
                              has finished reading the neighbours' rows), then
                              a barrier -- call before overwriting the slab, so
                              no neighbour still reads step s's boundary rows.

    (A device-side handshake with stream memory operations on IPC-shared
    counters was tried: on this driver a stream waiting on a counter that
    another stream writes never resumed, even inside one process -- DESIGN.md
    section 6.)  The slab must be written on the current stream before
    step()."""

    def __init__(self, slab: torch.Tensor, width: int, border=1, group=None):
        import ctypes

        from . import _capi

        self._capi, self._ct = _capi, ctypes
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if slab.dim() != 2 or slab.dtype != torch.int32 or not slab.is_cuda or \
                slab.stride(1) != 1:
            raise ValueError("slab must be a row-contiguous CUDA int32 [rows, S] tensor")
        self.slab, self.width, self.border = slab, int(width), border
        self.rows, self.stride = slab.shape[0], slab.stride(0)
        self.out = torch.empty_like(slab)
        self._opened = []
        self.above_ptr = self.below_ptr = None
        mine = (self._export(slab), self.rows, self.stride)
        everyone = [None] * self.world
        everyone[self.rank] = mine
        if self.world > 1:
            dist.all_gather_object(everyone, mine, group=group)
        if self.rank > 0:
            (h, off), rows, stride = everyone[self.rank - 1]
            self.above_ptr = self._open(h, off) + (rows - 1) * stride * 4
        if self.rank < self.world - 1:
            (h, off), _, _ = everyone[self.rank + 1]
            self.below_ptr = self._open(h, off)

    def _export(self, t: torch.Tensor):
        ct = self._ct
        handle = (ct.c_char * 64)()
        off = ct.c_int64()
        self._capi.call("be_ipc_export", ct.c_void_p(t.data_ptr()), handle, ct.byref(off))
        return bytes(handle), off.value

    def _open(self, handle: bytes, off: int) -> int:
        ptr = _ipc_open(self._capi, self._ct, handle, off)
        self._opened.append(handle)
        return ptr

    def _sync_all(self) -> None:
        if self.world > 1:
            torch.cuda.current_stream(self.slab.device).synchronize()
            dist.barrier(group=self.group)

    def acquire_for_write(self) -> None:
        """Return once every rank's kernel has finished reading its neighbours'
        rows (call before rewriting the slab)."""
        self._sync_all()

    def step(self) -> torch.Tensor:
        ct = self._ct
        from . import cuda as cu

        self._sync_all()                   # every slab of this step is complete
        st = ct.c_void_p(torch.cuda.current_stream(self.slab.device).cuda_stream)
        self._capi.call("be_edge_packed_halo_u32", ct.c_void_p(self.slab.data_ptr()),
                        ct.c_void_p(self.above_ptr) if self.above_ptr else None,
                        ct.c_void_p(self.below_ptr) if self.below_ptr else None,
                        ct.c_void_p(self.out.data_ptr()), self.rows, self.width, self.stride,
                        cu.fill_bit(self.border), 0, self.rows, st)
        return self.out

    def close(self):
        """Unmap the neighbours' buffers (after every rank's last step has
        finished reading, e.g. behind a barrier)."""
        for h in self._opened:
            _ipc_release(self._capi, self._ct, h)
        self._opened = []

"""Host-buffer batch API: the end-to-end path a user with data in host RAM calls.

`HostBatchEdges` runs a batch that lives in (pinned) host memory through the
device kernels in chunks, double-buffered over two CUDA streams so that the
host->device copy of one chunk overlaps the kernel and device->host copy of the
previous one (PCIe is full duplex; the kernel is ~100x faster than the link).
Only the packed result (1 bit per pixel) crosses back.
"""

from __future__ import annotations

import ctypes

import torch

from . import _capi
from . import cuda as cu


class HostBatchEdges:
    """Edges of a host batch: uint8 pixels [N, H, W] (kind='u8', fused pack)
    or packed int32 row words [N, H, S] (kind='packed', needs `width`).

    The chunk loop runs natively (`be_host_edges`, include/bitedge.h): chunk c
    is copied in, computed and copied out on stream c % 2, so the two copy
    directions and the kernels overlap without any per-chunk Python work."""

    def __init__(self, shape, kind: str = "u8", width: int | None = None, border=1,
                 chunk_images: int | None = None, device=None, chunk_rows: int | None = None,
                 halo_rows: tuple = (False, False), zero_copy: bool | None = None,
                 lanes: int = 3):
        """`halo_rows=(above, below)`: the host input of a single-image row slab
        also holds the row above its first row / below its last row (a row shard
        of a larger raster, multi-GPU); the result covers the slab's own rows.

        `zero_copy` (default: batches of up to 4 MiB of input, uint8 rows
        narrower than 1024 px): the kernel reads the page-locked host input and
        writes the page-locked host output over PCIe itself -- no copy
        operations, whose fixed latency dominates small batches (one 256^2 image:
        7 us against 20 us staged; scripts/zero_copy_rate.py).  Larger batches
        stream faster through the copy engines.  Buffers that are not
        page-locked always take the staged path."""
        if kind not in ("u8", "packed"):
            raise ValueError("kind must be 'u8' or 'packed'")
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        n, h, s = (int(v) for v in shape)
        self.kind, self.n, self.h = kind, n, h
        self.width = s if kind == "u8" else int(width)
        if kind == "packed" and s != cu.words_per_row(self.width, 32):
            raise ValueError("packed host rows must hold exactly ceil(width/32) words")
        self.border = border
        self.in_dtype = torch.uint8 if kind == "u8" else torch.int32
        self.halo_flags = (1 if halo_rows[0] else 0) | (2 if halo_rows[1] else 0)
        if self.halo_flags and n != 1:
            raise ValueError("halo_rows apply to a single image (n == 1)")
        self.in_shape = (n, h + bool(halo_rows[0]) + bool(halo_rows[1]), s)
        self.out_shape = (n, h, cu.words_per_row(self.width, 32))
        row_bytes = s * (1 if kind == "u8" else 4)
        per_img = h * row_bytes
        # a single image of >= 4 MiB: chunk it by rows (1-row halos; >= 4 chunks of
        # <= 8 MiB) so its copies overlap the kernels (be_host_edges_rows)
        self.rows_mode = n == 1 and chunk_images is None and (
            chunk_rows is not None or per_img >= (4 << 20) or self.halo_flags != 0)
        if chunk_rows is not None and not self.rows_mode:
            raise ValueError("chunk_rows applies to a single image (n == 1)")
        # submit() with several lanes moves a batch / image up to 64 / 128 MiB as
        # ONE chunk: consecutive batches then overlap their copies across the lanes
        # (C3 e2e 300 -> 321, C2 53.1 -> 53.9 Gpixel/s on one box), while a
        # blocking __call__ keeps the chunked pipeline inside the call
        whole_ok = lanes >= 2
        if self.rows_mode:
            auto = chunk_rows is None
            if auto:
                # two equal chunks up to 128 MiB images, then 64 MiB chunks: per-copy
                # fixed costs make small chunks slow (scripts/c3_e2e.py: C3 0.22 ms
                # at 2 x 4 MiB vs 0.27 at 4 x 2 MiB; C4 11.2 ms at 64 MiB chunks vs
                # 12.6 at 8 MiB)
                chunk_rows = max(1, min(64 << 20, -(-per_img // 2)) // row_bytes)
            self.chunk = int(chunk_rows)                                    # rows per chunk
            self.submit_chunk = h if (auto and whole_ok and per_img <= (128 << 20)) else self.chunk
            big = max(self.chunk, self.submit_chunk)
            self.d_in = [torch.empty((c + 2, s), dtype=self.in_dtype, device=self.device)
                         for c in (big, self.chunk)]
            self.d_out = [torch.empty((c, self.out_shape[2]), dtype=torch.int32,
                                      device=self.device) for c in (big, self.chunk)]
        else:
            auto = chunk_images is None
            if auto:
                # >= 8 MiB chunks, up to 64 MiB for big batches (fewer, larger copies)
                target = max(8 << 20, min(64 << 20, n * per_img // 8))
                chunk_images = max(1, min(n, target // max(1, per_img)))
            self.chunk = int(chunk_images)
            self.submit_chunk = n if (auto and whole_ok and n * per_img <= (64 << 20)) else self.chunk
            big = max(self.chunk, self.submit_chunk)
            self.d_in = [torch.empty((c, h, s), dtype=self.in_dtype, device=self.device)
                         for c in (big, self.chunk)]
            self.d_out = [torch.empty((c,) + self.out_shape[1:], dtype=torch.int32,
                                      device=self.device) for c in (big, self.chunk)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(2)]
        if zero_copy is None:
            zero_copy = (not self.rows_mode and n * per_img <= (4 << 20) and
                         (kind == "packed" or self.width < 1024))
        elif zero_copy and (self.rows_mode or (kind == "u8" and self.width >= 1024)):
            raise ValueError("zero_copy needs whole images and, for uint8, rows narrower "
                             "than 1024 px (the wider kernels stage rows with TMA)")
        self.zero_copy = bool(zero_copy)
        if lanes not in (1, 2, 3, 4):
            raise ValueError("lanes must be 1..4")
        self.lanes = 1 if self.zero_copy else lanes
        self.h2d_bytes = n * h * s * (1 if kind == "u8" else 4)
        if self.rows_mode:          # + the halo rows each chunk of a submit() copies in
            chunks = -(-h // self.submit_chunk)
            extra = 2 * (chunks - 1) + bool(self.halo_flags & 1) + bool(self.halo_flags & 2)
            self.h2d_bytes += extra * row_bytes
        self.d2h_bytes = n * self.out_shape[1] * self.out_shape[2] * 4
        P = ctypes.c_void_p
        self._din = (P * 2)(*[t.data_ptr() for t in self.d_in])
        self._dout = (P * 2)(*[t.data_ptr() for t in self.d_out])
        # submit() cycles through `lanes` lanes (buffers + stream pair): with one
        # lane, the next batch's first host->device copy waits in stream order for
        # the previous batch's device->host copies; with a lane per batch in
        # flight the copy engines of both directions run back to back (DESIGN 5).
        # Lanes past the first are allocated on first use.
        self._lanes = [(self.streams, self._din, self._dout)]
        self._keep = [self.d_in, self.d_out]
        self._adopt(self.streams, self.d_in + self.d_out)
        self._next = 0

    def _adopt(self, streams, bufs) -> None:
        """Hand caching-allocator blocks (allocated on the current stream) to the
        lane streams: the lane streams start after whatever the current stream
        queued before (the blocks may have been reused memory), and the blocks are
        recorded on them so the allocator never recycles one while a lane's copy
        or kernel is still queued."""
        cur = torch.cuda.current_stream(self.device)
        for st in streams:
            st.wait_stream(cur)
            for t in bufs:
                t.record_stream(st)

    def _lane(self, k: int):
        if k >= len(self._lanes):
            d_in = [torch.empty_like(t) for t in self.d_in]
            d_out = [torch.empty_like(t) for t in self.d_out]
            self._keep += [d_in, d_out]
            P = ctypes.c_void_p
            streams = [torch.cuda.Stream(self.device) for _ in range(2)]
            self._adopt(streams, d_in + d_out)
            self._lanes.append((streams, (P * 2)(*[t.data_ptr() for t in d_in]),
                                (P * 2)(*[t.data_ptr() for t in d_out])))
        return self._lanes[k]

    def new_host_buffers(self):
        hin = torch.empty(self.in_shape, dtype=self.in_dtype, pin_memory=True)
        hout = torch.empty(self.out_shape, dtype=torch.int32, pin_memory=True)
        return hin, hout

    def _check(self, host_in, host_out):
        if tuple(host_in.shape) != self.in_shape or host_in.dtype != self.in_dtype:
            raise ValueError(f"host input must be {self.in_dtype} {self.in_shape}")
        if host_in.is_cuda or not host_in.is_contiguous():
            raise ValueError("host input must be a contiguous CPU tensor (pinned for overlap)")
        if host_out is None:
            host_out = torch.empty(self.out_shape, dtype=torch.int32, pin_memory=True)
        if host_out.is_cuda or not host_out.is_contiguous() or tuple(host_out.shape) != self.out_shape:
            raise ValueError(f"host output must be a contiguous CPU int32 tensor {self.out_shape}")
        return host_out

    def _run(self, host_in, host_out, blocking: bool, lane: int = 0, chunk: int | None = None) -> None:
        P = ctypes.c_void_p
        streams, din, dout = self._lane(lane)
        chunk = self.chunk if chunk is None else chunk
        if self.zero_copy and host_in.is_pinned() and host_out.is_pinned():
            # one kernel over page-locked host memory (mapped: same address on the device)
            st = streams[0]
            wp = self.out_shape[2]
            if self.kind == "u8":
                _capi.call("be_pack_edge_u8", P(host_in.data_ptr()), P(host_out.data_ptr()),
                           self.n, self.h, self.width, self.width, wp, cu.fill_bit(self.border),
                           None, P(st.cuda_stream))
            else:
                _capi.call("be_edge_packed_u32", P(host_in.data_ptr()), P(host_out.data_ptr()),
                           self.n, self.h, self.width, wp, cu.fill_bit(self.border), 0,
                           P(st.cuda_stream))
            if blocking:
                st.synchronize()
            return
        if self.rows_mode:
            _capi.call("be_host_edges_rows", P(host_in.data_ptr()), 1 if self.kind == "u8" else 0,
                       P(host_out.data_ptr()), self.h, self.width, cu.fill_bit(self.border),
                       self.halo_flags, din, dout, chunk, P(streams[0].cuda_stream),
                       P(streams[1].cuda_stream), 1 if blocking else 0)
            return
        _capi.call("be_host_edges", P(host_in.data_ptr()), 1 if self.kind == "u8" else 0,
                   P(host_out.data_ptr()), self.n, self.h, self.width, cu.fill_bit(self.border),
                   din, dout, chunk, P(streams[0].cuda_stream),
                   P(streams[1].cuda_stream), 1 if blocking else 0)

    def __call__(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None,
                 sync: bool = True) -> torch.Tensor:
        """Run the batch, ordered after the caller's current stream; with
        sync=False the current stream is made to wait for the result and the
        host buffers must stay untouched until then."""
        host_out = self._check(host_in, host_out)
        cur = torch.cuda.current_stream(self.device)
        for s_ in self.streams:
            s_.wait_stream(cur)
        self._run(host_in, host_out, sync)
        if not sync:
            for s_ in self.streams:
                cur.wait_stream(s_)
        return host_out

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None) -> "Pending":
        """Enqueue the batch and return at once; the returned handle's
        `synchronize()` yields `host_out` when its last chunk has landed.

        Unlike `__call__(sync=False)` this does not tie the caller's stream to
        the batch, so consecutive submits pipeline across batches: the next
        batch's first host->device copy starts as soon as the copy engine is
        free instead of after this batch's last kernel and device->host copy.
        `host_in` must be ready on the host; both buffers must stay untouched
        until `synchronize()` returns."""
        host_out = self._check(host_in, host_out)
        lane = self._next
        self._next = (self._next + 1) % self.lanes
        zc = self.zero_copy and host_in.is_pinned() and host_out.is_pinned()
        self._run(host_in, host_out, False, lane, self.submit_chunk)
        evs = []
        # the zero-copy kernel runs on the lane's first stream only
        for s_ in self._lane(lane)[0][:1 if zc else 2]:
            e = torch.cuda.Event()
            e.record(s_)
            evs.append(e)
        return Pending(evs, host_out, self)


class Pending:
    """A submitted host batch (`HostBatchEdges.submit`).  Holds the pipe (and so
    its device buffers) until the batch is done."""

    def __init__(self, events, host_out, owner=None):
        self._events = events
        self.host_out = host_out
        self._owner = owner

    def query(self) -> bool:
        return all(e.query() for e in self._events)

    def synchronize(self) -> torch.Tensor:
        for e in self._events:
            e.synchronize()
        return self.host_out

    def wait(self, stream=None) -> None:
        """Make `stream` (default: the current one) wait for the batch."""
        stream = stream if stream is not None else torch.cuda.current_stream()
        for e in self._events:
            stream.wait_event(e)

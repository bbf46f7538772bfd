"""Host-buffer batch API: the end-to-end path a user with data in host RAM calls.

`HostBatchEdges` runs a batch that lives in (pinned) host memory through the
device kernels in chunks, double-buffered over three CUDA streams so that the
host->device copy of chunk c+1, the kernel of chunk c and the device->host
copy of chunk c-1 overlap (PCIe is full duplex; the kernel is ~100x faster
than the link).  Only the packed result (1 bit per pixel) crosses back.
"""

from __future__ import annotations

import torch

from . import cuda as cu


class HostBatchEdges:
    """Edges of a host batch: uint8 pixels [N, H, W] (kind='u8', fused pack)
    or packed int32 row words [N, H, S] (kind='packed', needs `width`)."""

    def __init__(self, shape, kind: str = "u8", width: int | None = None, border=1,
                 chunk_images: int | None = None, device=None):
        if kind not in ("u8", "packed"):
            raise ValueError("kind must be 'u8' or 'packed'")
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        n, h, s = (int(v) for v in shape)
        self.kind, self.n, self.h = kind, n, h
        self.width = s if kind == "u8" else int(width)
        self.border = border
        self.in_dtype = torch.uint8 if kind == "u8" else torch.int32
        self.in_shape = (n, h, s)
        self.out_shape = (n, h, cu.words_per_row(self.width, 32))
        if chunk_images is None:
            per_img = h * s * (1 if kind == "u8" else 4)
            chunk_images = max(1, min(n, (8 << 20) // max(1, per_img)))    # ~8 MiB per chunk
        self.chunk = int(chunk_images)
        self.d_in = [torch.empty((self.chunk, h, s), dtype=self.in_dtype, device=self.device)
                     for _ in range(2)]
        self.d_out = [torch.empty((self.chunk,) + self.out_shape[1:], dtype=torch.int32,
                                  device=self.device) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_k = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_k = [torch.cuda.Event() for _ in range(2)]
        self.ev_d2h = [torch.cuda.Event() for _ in range(2)]
        self.h2d_bytes = n * h * s * (1 if kind == "u8" else 4)
        self.d2h_bytes = n * self.out_shape[1] * self.out_shape[2] * 4

    def new_host_buffers(self):
        hin = torch.empty(self.in_shape, dtype=self.in_dtype, pin_memory=True)
        hout = torch.empty(self.out_shape, dtype=torch.int32, pin_memory=True)
        return hin, hout

    def __call__(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None,
                 sync: bool = True) -> torch.Tensor:
        if tuple(host_in.shape) != self.in_shape or host_in.dtype != self.in_dtype:
            raise ValueError(f"host input must be {self.in_dtype} {self.in_shape}")
        if host_out is None:
            host_out = torch.empty(self.out_shape, dtype=torch.int32, pin_memory=True)
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_k, self.s_d2h):
            s.wait_stream(cur)
        for c, lo in enumerate(range(0, self.n, self.chunk)):
            hi = min(self.n, lo + self.chunk)
            k = hi - lo
            b = c & 1
            din, dout = self.d_in[b][:k], self.d_out[b][:k]
            with torch.cuda.stream(self.s_h2d):
                if c >= 2:
                    self.s_h2d.wait_event(self.ev_k[b])       # kernel c-2 done reading d_in[b]
                din.copy_(host_in[lo:hi], non_blocking=True)
                self.ev_h2d[b].record(self.s_h2d)
            with torch.cuda.stream(self.s_k):
                self.s_k.wait_event(self.ev_h2d[b])
                if c >= 2:
                    self.s_k.wait_event(self.ev_d2h[b])       # d2h c-2 done reading d_out[b]
                if self.kind == "u8":
                    cu.pack_edges_u8(din, self.border, out=dout)
                else:
                    cu.edges_packed(din, self.width, self.border, out=dout)
                self.ev_k[b].record(self.s_k)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(self.ev_k[b])
                host_out[lo:hi].copy_(dout, non_blocking=True)
                self.ev_d2h[b].record(self.s_d2h)
        cur.wait_stream(self.s_d2h)
        if sync:
            self.s_d2h.synchronize()
        return host_out

"""HostBatchEdges lifetimes and stream ordering: a batch submitted
on a temporary pipe stays correct while the caching allocator churns on the
current stream, and lanes allocated lazily start after the current stream's
pending work."""

import numpy as np
import pytest

from oracle import cscan

pytestmark = pytest.mark.gpu


def test_submit_on_temporary_pipe(cuda_dev):
    import torch

    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.host import HostBatchEdges

    imgs = synth.c2_images(512)
    exp = cscan.scan_u8(imgs.numpy(), 1)
    hin = torch.empty(tuple(imgs.shape), dtype=torch.uint8, pin_memory=True)
    hin.copy_(imgs)
    pend = []
    for k in range(3):
        hout = torch.empty((512, 64, 2), dtype=torch.int32, pin_memory=True)
        # zero_copy off: the staged path owns device buffers on the lane streams
        pend.append(HostBatchEdges(tuple(imgs.shape), zero_copy=False).submit(hin, hout))
        # churn: the freed pipe's blocks would be handed out again right here
        for _ in range(8):
            torch.empty(8 << 20, dtype=torch.uint8, device=cuda_dev).fill_(0xAB)
    for p in pend:
        assert (p.synchronize().numpy().view(np.uint32) == exp).all()


def test_lazy_lanes_after_pending_work(cuda_dev):
    import torch

    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.host import HostBatchEdges

    imgs = synth.c2_images(256)
    exp = cscan.scan_u8(imgs.numpy(), 1)
    hin = torch.empty(tuple(imgs.shape), dtype=torch.uint8, pin_memory=True)
    hin.copy_(imgs)
    pipe = HostBatchEdges(tuple(imgs.shape), zero_copy=False, lanes=3)
    outs = [torch.empty((256, 64, 2), dtype=torch.int32, pin_memory=True) for _ in range(6)]
    pend = []
    for k in range(6):
        torch.cuda._sleep(200_000)                 # pending current-stream work
        pend.append(pipe.submit(hin, outs[k]))
    for p in pend:
        assert (p.synchronize().numpy().view(np.uint32) == exp).all()

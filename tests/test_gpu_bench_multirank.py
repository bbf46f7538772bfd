"""bench.py's multi-rank paths (torchrun, 2 ranks) exercised on ONE GPU:
BITEDGE_SHARE_GPU puts both ranks on device 0 and BITEDGE_DIST_BACKEND=gloo
replaces NCCL (which refuses two ranks per device).  Functional only -- the
numbers of such a run mean nothing; the real multi-GPU run is the driver's."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra", [["--config", "c2", "--steps", "300"],
                                   ["--config", "c4", "--steps", "4"],
                                   ["--config", "c4", "--steps", "4", "--no-e2e", "--halo", "nccl"]],
                         ids=["c2-batch", "c4-rows-p2p", "c4-rows-nccl"])
def test_bench_two_ranks_one_gpu(extra, cuda_dev):
    if "nccl" in extra:
        pytest.skip("NCCL halos need two devices (gloo has no CUDA send/recv)")
    env = dict(os.environ, BITEDGE_SHARE_GPU="1", BITEDGE_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--warmup", "3", *extra]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity"]["ok"]
    if "c4" in extra:
        assert d["scaling"] == "strong" and "p2p" in d["config"]["parallelism"]
        # e2e of the row shards (host halos): both ranks' slabs plus their halo rows
        assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > (65536 * 2048 * 4)
    else:
        assert d["scaling"] == "weak" and d["config"]["global_batch"] == 8192

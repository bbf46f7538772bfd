"""bench.py's multi-rank paths (torchrun, 2 ranks) exercised on ONE GPU:
BITEDGE_SHARE_GPU puts both ranks on device 0 and BITEDGE_DIST_BACKEND=gloo
replaces NCCL (which refuses two ranks per device).  Functional only -- the
numbers of such a run mean nothing; the real multi-GPU run is the driver's."""

import json
import os
import signal
import socket
import subprocess
import sys
import time

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(args, env, world, timeout):
    """Launch the `world` ranks of `python bench.py args` directly (what torchrun
    does: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* in the environment), each in
    its own session, and kill every rank on timeout -- torchrun starts its
    workers in new sessions, so killing a timed-out torchrun would leave its
    ranks running on the GPU.  Returns rank 0's CompletedProcess; the other
    ranks' stderr is appended to it on failure."""
    port = str(_port())
    procs = []
    for r in range(world):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(world), LOCAL_WORLD_SIZE=str(world),
                 MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, "bench.py", *args], cwd=ROOT, env=e,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                                      start_new_session=True))
    deadline = time.time() + timeout
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=max(1.0, deadline - time.time())))
    except subprocess.TimeoutExpired:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, signal.SIGKILL)
        errs = [p.communicate()[1] for p in procs]
        pytest.fail(f"timed out after {timeout} s: bench.py {' '.join(args)}\n" +
                    "\n".join(e[-2000:] for e in errs))
    rc = max(p.returncode for p in procs)
    err = "\n".join(f"[rank {r}] {o[1][-2000:]}" for r, o in enumerate(outs)) if rc else outs[0][1]
    return subprocess.CompletedProcess(args, rc, outs[0][0], err)


@pytest.mark.parametrize("extra", [["--config", "c2", "--steps", "300"],
                                   ["--config", "c2", "--steps", "300", "--weak"],
                                   ["--config", "c4", "--steps", "4"],
                                   ["--config", "c4", "--steps", "4", "--halo", "p2p"]],
                         ids=["c2-strong", "c2-weak", "c4-rows-nccl-path", "c4-rows-p2p"])
def test_bench_two_ranks_one_gpu(extra, cuda_dev):
    """The NCCL halo path runs RowShardedEdges on CUDA with gloo standing in for
    NCCL (rows staged through the host); p2p runs the IPC peer reads with the
    device-side handshake."""
    env = dict(os.environ, BITEDGE_SHARE_GPU="1", BITEDGE_DIST_BACKEND="gloo")
    res = _run_ranks(["--gpus", "2", "--warmup", "3", "--no-dropin", *extra], env, 2, timeout=300)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity"]["ok"]
    assert d["parity"]["ranks"] == 2
    if "c4" in extra:
        assert d["scaling"] == "strong" and "row-shard x2" in d["config"]["parallelism"]
        assert ("p2p" if "p2p" in extra else "nccl") in d["method"]["halo"]
        assert "per-iteration barrier" in d["method"]["timing"]
        assert d["parity"]["checked_px"] == 65536 * 65536
        # e2e of the row shards (host halos): both ranks' slabs plus their halo rows
        assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > (65536 * 2048 * 4)
    elif "--weak" in extra:
        assert d["scaling"] == "weak" and d["config"]["global_batch"] == 8192
    else:
        assert d["scaling"] == "strong" and d["config"]["global_batch"] == 4096
        assert d["parity"]["checked_px"] == 4096 * 64 * 64

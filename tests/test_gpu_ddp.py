"""SESGDDataParallel (gradient fusion buffer + backward/sync overlap) on 1, 2 and
(if present) 4 GPUs: every training step's result equals the CPU oracle's step replayed on the
gradients autograd produced, bit for bit, and with overlap on every bucket's sync was enqueued
from a gradient hook inside backward."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, gpus, m, overlap=1, mode=0, iters=4, static=0):
    if not torch.cuda.is_available() or torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    out = str(tmp_path / "log.npy")
    for _attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
               os.path.join(ROOT, "tests", "ddp_worker.py"), "--gsize", str(m), "--iters", str(iters),
               "--overlap", str(overlap), "--mode", str(mode), "--static", str(static), "--out", out]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        if "EADDRINUSE" not in res.stderr:
            break
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    log = np.load(out)
    assert log.shape == (iters, 7)
    assert np.all(log[:, 2] == 0), f"x differs from the oracle replay: {log}"
    assert np.all(log[:, 3] == 0), f"v differs from the oracle replay: {log}"
    assert np.all(log[:, 5] > 0), "no gradient reached the fusion buffer"
    return log


def test_ddp_one_gpu_local_sgd(tmp_path):
    log = _run(tmp_path, 1, 1)
    assert np.all(log[:, 4] == 3), "buckets not launched from the gradient hooks"
    assert np.all(log[:, 6] == 6)  # one hook per parameter
    assert log[-1, 1] < log[0, 1] * 1.5


@pytest.mark.multigpu
@pytest.mark.parametrize("mode", [0, 1])
def test_ddp_two_gpus_overlap(tmp_path, mode):
    log = _run(tmp_path, 2, 2, mode=mode)
    assert np.all(log[:, 4] == 3)


@pytest.mark.multigpu
def test_ddp_two_gpus_no_overlap(tmp_path):
    log = _run(tmp_path, 2, 2, overlap=0)
    assert np.all(log[:, 4] == 0)
    assert np.all(log[:, 6] == 0)  # no hooks at all


@pytest.mark.multigpu
def test_ddp_two_gpus_static_graph(tmp_path):
    """static_graph: 6 hooks (one per parameter) in step 0, trimmed at its end to one per bucket;
    every bucket still launches from backward and every step still equals the oracle replay."""
    log = _run(tmp_path, 2, 2, static=1, iters=5)
    assert np.all(log[:, 4] == 3)
    assert np.all(log[:, 6] == 3)


def test_ddp_one_gpu_static_graph(tmp_path):
    log = _run(tmp_path, 1, 1, static=1, iters=4)
    assert np.all(log[:, 4] == 3)


@pytest.mark.multigpu
@pytest.mark.parametrize("m", [2, 4])
def test_ddp_four_gpus(tmp_path, m):
    log = _run(tmp_path, 4, m, iters=6)
    assert np.all(log[:, 4] == 3)

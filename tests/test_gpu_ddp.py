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


def _run(tmp_path, gpus, m, overlap=1, mode=0, iters=4, static=0, graph=0):
    if not torch.cuda.is_available() or torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    out = str(tmp_path / "log.npy")
    for _attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
               os.path.join(ROOT, "tests", "ddp_worker.py"), "--gsize", str(m), "--iters", str(iters),
               "--overlap", str(overlap), "--mode", str(mode), "--static", str(static), "--graph", str(graph),
               "--out", out]
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


@pytest.mark.multigpu
@pytest.mark.parametrize("gpus,static", [(2, 1), (4, 0)])
def test_ddp_captured_training_step_multigpu(tmp_path, gpus, static):
    """one process per GPU: from step 2 on, the whole training step is ONE replayed CUDA graph
    (SESGDDataParallel.enable_graphs), every step still equal to the oracle's replay"""
    _run(tmp_path, gpus, 2, static=static, iters=6, graph=1)


def test_ddp_one_gpu_static_graph(tmp_path):
    log = _run(tmp_path, 1, 1, static=1, iters=4)
    assert np.all(log[:, 4] == 3)


@pytest.mark.multigpu
@pytest.mark.parametrize("m", [2, 4])
def test_ddp_four_gpus(tmp_path, m):
    log = _run(tmp_path, 4, m, iters=6)
    assert np.all(log[:, 4] == 3)


# ---------------------------------------------------------------- loopback: R replicas on one GPU
@pytest.mark.parametrize("world,m,mode,static", [(2, 2, 0, 0), (4, 2, 0, 1), (4, 4, 1, 0)])
def test_ddp_loopback_replicas(world, m, mode, static):
    """SESGDDataParallel on loopback virtual ranks: `world` model replicas in ONE process on ONE GPU,
    each on an engine.LoopbackGroup rank (the NVLink-path kernel, K4W), distinct random inits made
    equal by copying replica 0's fusion buffer (what the process-group broadcast does), the bucket
    syncs enqueued from gradient hooks during each replica's backward; every step equals the oracle's
    step replayed on the gradients autograd produced, bit for bit"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.nn.functional as F

    import oracle
    from paper_2007_00433_b200 import sesgd as C
    from paper_2007_00433_b200.ddp import SESGDDataParallel
    from paper_2007_00433_b200.engine import LoopbackGroup
    from paper_2007_00433_b200.workloads import assign_buckets
    LR, MU = 0.05, 0.9
    dev = torch.device("cuda", 0)

    def mlp(seed):
        torch.manual_seed(seed)
        return torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 512),
                                   torch.nn.ReLU(), torch.nn.Linear(512, 10)).to(dev)

    models = [mlp(r) for r in range(world)]
    # load every forward / backward kernel once before any virtual rank's exchange kernel spins:
    # with CUDA's lazy module loading, a first-use load behind a spinning grid on the same GPU can
    # stall until the peer timeout (one process per GPU never has that)
    warm = mlp(99)
    F.cross_entropy(warm(torch.randn(64, 256, device=dev)), torch.randint(0, 10, (64,), device=dev)).backward()
    torch.cuda.synchronize()
    sizes = [p.numel() for p in models[0].parameters()]
    caps = dict(first_bucket_bytes=16 << 10, bucket_bytes=256 << 10)
    bsizes = [sum(sizes[i] for i in b) for b in assign_buckets(sizes, caps["first_bucket_bytes"], caps["bucket_bytes"])]
    grp = LoopbackGroup(world, world, m, bsizes, seed=42, mode=mode, timeout_ms=20000)
    ddps = [SESGDDataParallel(models[r], world, m, lr=LR, momentum=MU, rank=r, world=world, engine=grp[r],
                              static_graph=bool(static), **caps) for r in range(world)]
    with torch.no_grad():  # Alg.1 line 1: the same x_0 everywhere
        for r in range(1, world):
            grp[r].x_flat[0].copy_(grp[0].x_flat[0])
    torch.cuda.synchronize()
    for t in range(4):
        X0 = np.stack([e.x_flat[0].cpu().numpy() for e in grp])
        V0 = np.stack([e.v_flat[0].cpu().numpy() for e in grp])
        in_bwd = []
        for r, (model, ddp) in enumerate(zip(models, ddps)):
            gen = torch.Generator(device=dev).manual_seed(1000 * t + r)
            inp = torch.randn(64, 256, device=dev, generator=gen)
            lab = torch.randint(0, 10, (64,), device=dev, generator=gen)
            ddp.begin_step(t)
            F.cross_entropy(model(inp), lab).backward()
            in_bwd.append(ddp.launched_in_backward)
        for ddp in ddps:
            ddp.finish_step()
        torch.cuda.synchronize()
        grp.poll()
        G = np.stack([e.g_flat[0].cpu().numpy() for e in grp])
        X1 = np.stack([e.x_flat[0].cpu().numpy() for e in grp])
        V1 = np.stack([e.v_flat[0].cpu().numpy() for e in grp])
        assert np.abs(G).max() > 0
        assert all(k >= len(bsizes) - 1 for k in in_bwd), in_bwd  # synced from hooks, inside backward
        _, canon, _ = oracle.groups(42, t, world, m)
        x, v = X0.copy(), V0.copy()
        oracle.step(world, m, canon, x, v, G, LR, MU, mode)
        assert np.array_equal(x.view(np.uint32), X1.view(np.uint32)), t
        assert np.array_equal(v.view(np.uint32), V1.view(np.uint32)), t
    for ddp in ddps:
        ddp.close()
    grp.close()


@pytest.mark.parametrize("world,m,static", [(2, 2, 1), (4, 2, 0)])
def test_ddp_loopback_captured_training_step(world, m, static):
    """A whole SESGDDataParallel training step -- zero grads, device-side begin_iter, forward,
    backward with the bucket syncs launched from gradient hooks on the side stream, finish -- captured
    ONCE per replica with torch.cuda.graph (device-resident iterations) and replayed for 4 steps on
    loopback virtual ranks: every replayed step equals the oracle's step on the gradients it produced"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.nn.functional as F

    import oracle
    from paper_2007_00433_b200.ddp import SESGDDataParallel
    from paper_2007_00433_b200.engine import LoopbackGroup
    from paper_2007_00433_b200.workloads import assign_buckets
    LR, MU = 0.05, 0.9
    dev = torch.device("cuda", 0)

    def mlp(seed):
        torch.manual_seed(seed)
        return torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 10)).to(dev)

    warm = mlp(99)
    F.cross_entropy(warm(torch.randn(64, 256, device=dev)), torch.randint(0, 10, (64,), device=dev)).backward()
    torch.cuda.synchronize()
    models = [mlp(r) for r in range(world)]
    sizes = [p.numel() for p in models[0].parameters()]
    caps = dict(first_bucket_bytes=16 << 10, bucket_bytes=256 << 10)
    bsizes = [sum(sizes[i] for i in b) for b in assign_buckets(sizes, caps["first_bucket_bytes"], caps["bucket_bytes"])]
    grp = LoopbackGroup(world, world, m, bsizes, seed=42, timeout_ms=20000)
    ddps = [SESGDDataParallel(models[r], world, m, lr=LR, momentum=MU, rank=r, world=world, engine=grp[r],
                              static_graph=bool(static), **caps) for r in range(world)]
    with torch.no_grad():
        for r in range(1, world):
            grp[r].x_flat[0].copy_(grp[0].x_flat[0])
    inp = [torch.zeros(64, 256, device=dev) for _ in range(world)]
    lab = [torch.zeros(64, dtype=torch.long, device=dev) for _ in range(world)]

    def feed(t):
        for r in range(world):
            gen = torch.Generator(device=dev).manual_seed(1000 * t + r)
            inp[r].copy_(torch.randn(64, 256, device=dev, generator=gen))
            lab[r].copy_(torch.randint(0, 10, (64,), device=dev, generator=gen))

    def check(t, X0, V0):
        torch.cuda.synchronize()
        grp.poll()
        G = np.stack([e.g_flat[0].cpu().numpy() for e in grp])
        X1 = np.stack([e.x_flat[0].cpu().numpy() for e in grp])
        V1 = np.stack([e.v_flat[0].cpu().numpy() for e in grp])
        assert np.abs(G).max() > 0
        _, canon, _ = oracle.groups(42, t, world, m)
        x, v = X0.copy(), V0.copy()
        oracle.step(world, m, canon, x, v, G, LR, MU, 0)
        assert np.array_equal(x.view(np.uint32), X1.view(np.uint32)), t
        assert np.array_equal(v.view(np.uint32), V1.view(np.uint32)), t

    def state():
        torch.cuda.synchronize()
        return (np.stack([e.x_flat[0].cpu().numpy() for e in grp]), np.stack([e.v_flat[0].cpu().numpy() for e in grp]))

    T_eager = 2
    for t in range(T_eager):  # eager warm-up steps (host iterations; static_graph trims the hooks)
        feed(t)
        X0, V0 = state()
        for r in range(world):
            ddps[r].begin_step(t)
            F.cross_entropy(models[r](inp[r]), lab[r]).backward()
        for d in ddps:
            d.finish_step()
        check(t, X0, V0)
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    graphs = []
    for r in range(world):
        ddps[r].enable_graphs()
        g = torch.cuda.CUDAGraph()
        streams[r].wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=streams[r]):
            ddps[r].begin_step()
            F.cross_entropy(models[r](inp[r]), lab[r]).backward()
            ddps[r].finish_step()
        graphs.append(g)
    for t in range(T_eager, T_eager + 4):
        feed(t)
        X0, V0 = state()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                graphs[r].replay()
        check(t, X0, V0)
    for d in ddps:
        d.close()
    grp.close()

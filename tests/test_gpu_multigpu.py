"""Multi-GPU parity of the NVLink P2P paths (K3 one-shot, K4 two-shot, K5 ring) against the CPU oracle.

Every test runs over two transports:
* ``loopback`` -- the R ranks are virtual ranks on ONE GPU (engine.LoopbackGroup: R contexts, each
  with its own workspace and stream and SMs / R of the device, attached to each other with
  sesgd_attach_peers), so the multi-GPU kernels, their flags, stage / receive slots and reuse
  guards run on a 1-GPU box;
* ``nvlink`` -- tests/mgpu_worker.py under torch.distributed.run, one process per GPU over
  NVLink / NVSwitch (skipped on boxes with fewer GPUs).
Both compare every worker's x, v after T iterations with the oracle on the same seeded inputs.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_TRANSPORT = "loopback"


@pytest.fixture(autouse=True, params=["loopback", pytest.param("nvlink", marks=pytest.mark.multigpu)])
def transport(request):
    global _TRANSPORT
    _TRANSPORT = request.param
    yield request.param


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(tmp_path, gpus, n, m, T, buckets, mode=0, t0=0, grid=0, variant=-1, fused=1, batch=0,
            lag=0, path=0, hop_ns=0, tma=0, period=1, final_avg=0, schedule=0, consensus=0, wd=0.0,
            bf16=0, coords=None, protocol=-1, release_every=0, devit=0, hybrid=0):
    """`gpus` ranks: processes on as many GPUs (nvlink) or virtual ranks on cuda:0 (loopback)"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    loop = _TRANSPORT == "loopback"
    if not loop and torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    out = str(tmp_path / "res")
    extra = []
    if coords is not None:
        np.save(str(tmp_path / "coords.npy"), np.asarray(coords, np.int64))
        extra = ["--coords", str(tmp_path / "coords.npy")]
    for _attempt in range(3):  # the rendezvous port can be taken between probe and bind
        launcher = ([sys.executable] if loop else
                    [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
                     "--master-addr=127.0.0.1", f"--master-port={_free_port()}"])
        cmd = [*launcher,
               os.path.join(ROOT, "tests", "mgpu_worker.py"), "--workers", str(n), "--gsize", str(m),
               "--iters", str(T), "--buckets", ",".join(map(str, buckets)), "--mode", str(mode),
               "--t0", str(t0), "--grid", str(grid), "--variant", str(variant), "--fused", str(fused),
               "--batch", str(batch), "--lag", str(lag), "--path", str(path), "--hop-ns", str(hop_ns),
               "--tma", str(tma), "--period", str(period), "--final-avg", str(final_avg),
               "--schedule", str(schedule), "--consensus", str(consensus), "--wd", repr(wd),
               "--bf16", str(bf16), "--protocol", str(protocol), "--release-every", str(release_every), "--devit", str(devit), "--hybrid", str(hybrid), "--loopback", str(gpus if loop else 0), *extra,
               "--out", out]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        if "EADDRINUSE" not in res.stderr:
            break
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    X = np.zeros((n, sum(buckets) if coords is None else len(coords)), np.float32)
    V = np.zeros_like(X)
    for r in range(gpus):
        d = np.load(f"{out}.rank{r}.npz")
        X[d["workers"]] = d["X"]
        V[d["workers"]] = d["V"]
    return X, V


def _oracle(n, m, L, T, mode, t0=0, coords=None):
    x = np.tile(synth.x0_host(L, coords=coords), (n, 1))
    v = np.zeros_like(x)
    oracle.run(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, mode=mode, t0=t0, coords=coords)
    return x, v


def _sample(buckets, k=3000, seed=11):
    """bucket edges and ragged tails plus random interior coordinates (global element indices)"""
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]])
    edges = np.concatenate([[o, o + 1, o + s - 1, o + s - 2] for o, s in zip(offs, buckets)])
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([edges, rng.integers(0, sum(buckets), k - len(edges))])).astype(np.int64)


@pytest.mark.parametrize("gpus", [8, 4, 2])
def test_resnet50_bench_shape_full_size(tmp_path, gpus):
    """BASELINE configs[1] at full size in bench.py's launch configuration: n = 8, group_size 2, the
    five ResNet-50 DDP buckets (25,557,032 fp32), T = 100, one fused launch per iteration on every
    rank; gpus = 8 is the north star's one worker per GPU (K4), 4 and 2 the bench's N = 4 / N = 2
    lines (2 and 4 workers per GPU, the MULTI K4).  The oracle replays ~3000 sampled coordinates."""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    buckets = list(RESNET50_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, gpus, 8, 2, 100, buckets, coords=coords)
    x, v = _oracle(8, 2, sum(buckets), 100, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


def test_vgg16_cfg3_shape_full_size(tmp_path):
    """BASELINE configs[2] at full size: n = 16 workers, 2 per GPU on 8 ranks, group_size 4 (groups
    span 1-4 ranks), the six VGG-16 DDP buckets (138,357,544 fp32), 10 iterations, MULTI K4;
    sampled coordinates against the oracle."""
    from paper_2007_00433_b200.workloads import VGG16_BUCKETS
    buckets = list(VGG16_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, 8, 16, 4, 10, buckets, coords=coords)
    x, v = _oracle(16, 4, sum(buckets), 10, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


def _compare(got, want):
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-7)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_one_worker_each(tmp_path, mode, fused):
    """n=2 (group_size=2 = n: full averaging, Ring-SGD special case) across 2 GPUs through the
    one-shot kernel (K3), one fused launch over all buckets (sesgd_sync_all) or one per bucket."""
    buckets = [100003, 7, 40000]
    X, V = _launch(tmp_path, 2, 2, 2, 6, buckets, mode, fused=fused, path=2)
    x, v = _oracle(2, 2, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("path,protocol", [(2, -1), (4, 0), (4, 1)])
@pytest.mark.parametrize("n,m", [(4, 2), (8, 2), (8, 4), (4, 1), (8, 8)])
def test_two_gpus_resident_pairs(tmp_path, n, m, path, protocol):
    """n/2 workers per GPU through K3 (one-shot) and K4 (two-shot): groups mix co-resident
    members (read in place from the local stage, updated in place) and remote members (NVLink
    push); all-local groups are updated in registers; the schedule changes every iteration,
    exercising the call-2 receive-slot guard."""
    buckets = [65537, 3, 20000]
    T = 7
    X, V = _launch(tmp_path, 2, n, m, T, buckets, path=path, protocol=protocol)
    x, v = _oracle(n, m, sum(buckets), T, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("protocol", [0, 1])
@pytest.mark.parametrize("n,m", [(8, 4), (4, 2)])
def test_two_gpus_resident_pairs_twoshot_grad(tmp_path, n, m, protocol):
    """K4 with co-resident members in GRAD mode: the slice owner applies the mean gradient to
    its co-resident members' v and x."""
    buckets = [65537, 3, 20000]
    X, V = _launch(tmp_path, 2, n, m, 6, buckets, mode=1, path=4, protocol=protocol)
    x, v = _oracle(n, m, sum(buckets), 6, 1)
    _compare(X, x)
    _compare(V, v)


def test_two_gpus_small_grid_many_chunks(tmp_path):
    """A small grid forces many chunks per CTA (epoch sequence k > 0 within a launch)."""
    buckets = [300001]
    X, V = _launch(tmp_path, 2, 4, 2, 5, buckets, grid=8)
    x, v = _oracle(4, 2, sum(buckets), 5, 0)
    _compare(X, x)


@pytest.mark.parametrize("variant,batch,lag", [(0, 1, 1), (0, 1, 5), (1, 1, 1), (8, 4, 2), (32, 16, 4),
                                               (10, 64, 16), (3, 2, 8)])
def test_two_gpus_kernel_variants(tmp_path, variant, batch, lag):
    """COMM CTAs x chunks per release x fold lag: every pipeline shape gives the oracle's
    bits, with a small grid so each CTA pipelines several chunks."""
    buckets = [250001, 13, 70000]
    X, V = _launch(tmp_path, 2, 4, 2, 5, buckets, grid=24, variant=variant, batch=batch, lag=lag)
    x, v = _oracle(4, 2, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


def test_two_gpus_random_access_resume(tmp_path):
    """begin_iter at t0 = 1000 (resume): the flags are keyed by call index, not t."""
    buckets = [90001]
    X, V = _launch(tmp_path, 2, 4, 2, 4, buckets, t0=1000)
    x, v = _oracle(4, 2, sum(buckets), 4, 0, t0=1000)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("path", [2, 4])
def test_four_gpus(tmp_path, path):
    buckets = [200003, 5000]
    X, V = _launch(tmp_path, 4, 8, 4, 6, buckets, path=path)
    x, v = _oracle(8, 4, sum(buckets), 6, 0)
    _compare(X, x)
    _compare(V, v)


def test_four_gpus_sixteen_workers_twoshot(tmp_path):
    """BASELINE cfg 3's shape on 4 GPUs: n = 16, m = 4, four workers per GPU (groups span 1-4
    GPUs), K4 two-shot."""
    buckets = [100003, 77]
    X, V = _launch(tmp_path, 4, 16, 4, 5, buckets, path=4)
    x, v = _oracle(16, 4, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


def _oracle_ring(n, m, buckets, T, mode):
    """ring-order oracle, bucket by bucket (each bucket is sliced separately)"""
    X, V, e0 = [], [], 0
    for L in buckets:
        x = np.tile(synth.x0_host(L, e0=e0), (n, 1))
        v = np.zeros_like(x)
        oracle.run_ring(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, mode=mode, e0=e0)
        X.append(x)
        V.append(v)
        e0 += L
    return np.concatenate(X, axis=1), np.concatenate(V, axis=1)


@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_ring_path(tmp_path, mode):
    """K5 (the paper's Ring-AllReduce inside the group, 2(m-1) handshakes) on 2 GPUs, m = n = 2:
    ring order equals the ascending fold for two members, so it matches both oracles bit-exactly."""
    buckets = [100003, 9, 4096]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, mode, path=3)
    x, v = _oracle(2, 2, sum(buckets), 5, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m", [2, 4])
def test_four_gpus_ring_path(tmp_path, m):
    """K5 on 4 GPUs: m = 4 is the Ring-SGD special case (ring over all workers, 6 handshakes);
    bit-exact against the ring-order oracle, within the north-star tolerance of the fold."""
    buckets = [70001, 33]
    X, V = _launch(tmp_path, 4, 4, m, 4, buckets, path=3)
    xr, vr = _oracle_ring(4, m, buckets, 4, 0)
    _compare(X, xr)
    _compare(V, vr)
    x, _ = _oracle(4, m, sum(buckets), 4, 0)
    np.testing.assert_allclose(X, x, rtol=1e-5, atol=1e-7)


def test_two_gpus_ring_path_injected_latency(tmp_path):
    """The injected per-hop delay changes only the timing, never the bits."""
    buckets = [20000]
    X, V = _launch(tmp_path, 2, 2, 2, 3, buckets, path=3, hop_ns=100000)
    x, v = _oracle(2, 2, sum(buckets), 3, 0)
    _compare(X, x)


# ---------------------------------------------------------------- K4 two-shot (path 4)
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_twoshot(tmp_path, mode, fused):
    """K4 with the epoch-flag protocol (SESGD_OPT_PROTOCOL 0: reduce-scatter + all-gather pushes,
    two handshake rounds, fence + flags) on 2 GPUs, n = m = 2: the slice owner folds in ascending
    worker id and divides once, so the bits are the oracle's."""
    buckets = [100003, 7, 40000, 4096]
    X, V = _launch(tmp_path, 2, 2, 2, 6, buckets, mode, fused=fused, path=4, protocol=0)
    x, v = _oracle(2, 2, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("lag,grid", [(1, 8), (2, 24), (3, 0), (8, 16), (64, 4)])
def test_two_gpus_twoshot_pipeline_shapes(tmp_path, lag, grid):
    """Small grids (many chunks per CTA) x fold lags (1 .. 32 per round): every pipeline depth,
    including ones longer than a CTA's chunk list, gives the oracle's bits (flag protocol)."""
    buckets = [250001, 13, 70000]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, grid=grid, lag=lag, path=4, protocol=0)
    x, v = _oracle(2, 2, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


def test_two_gpus_twoshot_resume(tmp_path):
    buckets = [90001]
    X, V = _launch(tmp_path, 2, 2, 2, 4, buckets, t0=1000, path=4)
    x, v = _oracle(2, 2, sum(buckets), 4, 0, t0=1000)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("mode", [0, 1])
def test_four_gpus_twoshot(tmp_path, m, mode):
    """K4 (flag protocol) on 4 GPUs: m = 2 (groups change every iteration) and m = 4 (4 slice
    owners, ragged last slice and bucket tails)."""
    buckets = [200003, 5000, 1]
    X, V = _launch(tmp_path, 4, 4, m, 6, buckets, mode, path=4, protocol=0)
    x, v = _oracle(4, m, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("lag,grid", [(0, 0), (1, 8), (6, 24), (64, 4)])
def test_two_gpus_twoshot_tma(tmp_path, mode, lag, grid):
    """K4 with TMA bulk pushes (SESGD_OPT_PUSH_TMA): shared-memory chunk images sent with
    cp.async.bulk, flags released after the bulk groups complete; ragged tails by plain stores."""
    buckets = [250001, 13, 70000, 3]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, mode, grid=grid, lag=lag, path=4, tma=1)
    x, v = _oracle(2, 2, sum(buckets), 5, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m", [2, 4])
def test_four_gpus_twoshot_tma(tmp_path, m):
    buckets = [200003, 5000, 1]
    X, V = _launch(tmp_path, 4, 4, m, 6, buckets, 0, path=4, tma=1)
    x, v = _oracle(4, m, sum(buckets), 6, 0)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- NEXT-2: Local-SESGD + final average
@pytest.mark.parametrize("path", [2, 4])
@pytest.mark.parametrize("n,m,period", [(4, 2, 2), (2, 2, 3), (4, 4, 2)])
def test_two_gpus_local_sesgd_final_average(tmp_path, n, m, period, path):
    """Local-SESGD (exchange only when (t + 1) % period == 0; m = n is Local-SGD) over NVLink,
    then Algorithm 1's final global average (one two-shot exchange with group_size = n on a
    zero-momentum context, lr = 0): the oracle's bits (its ascending fold over all n workers)."""
    buckets = [65537, 3, 20000]
    T = 5
    X, V = _launch(tmp_path, 2, n, m, T, buckets, path=path, period=period, final_avg=1)
    x = np.tile(synth.x0_host(sum(buckets)), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=period)
    _compare(V, v)
    _compare(X, oracle.global_average(x))


@pytest.mark.parametrize("gpus,n,m", [(2, 4, 2), (2, 8, 4), (4, 8, 2)])
def test_dimension_exchange_schedule_multigpu(tmp_path, gpus, n, m):
    """NEXT-3 over NVLink (K4): Stone's dimension-exchange schedule, the oracle's bits."""
    buckets = [65537, 3]
    T = 6
    X, V = _launch(tmp_path, gpus, n, m, T, buckets, schedule=1)
    x = np.tile(synth.x0_host(sum(buckets)), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1,
                     schedule=oracle.SCHED_STONE)
    _compare(X, x)
    _compare(V, v)


def test_two_gpus_consensus_metric(tmp_path):
    """NEXT-4 across GPUs: all-gathered rows + K9 on every rank equal the oracle's metric."""
    buckets = [65537, 3]
    n, m, T = 4, 2, 6
    _launch(tmp_path, 2, n, m, T, buckets, consensus=1)
    x, _ = _oracle(n, m, sum(buckets), T, 0)
    oss, omx = oracle.consensus(x)
    for r in range(2):
        ss, mx = np.load(str(tmp_path / "res") + f".rank{r}.npz")["cons"]
        assert abs(ss - oss) <= 1e-9 * oss and abs(mx - omx) <= 1e-12 * omx


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n,path", [(4, 4), (4, 2), (2, 3), (2, 4)])
def test_two_gpus_weight_decay(tmp_path, n, path, mode):
    """NEXT-4 over NVLink: weight decay in K4 (two-shot), K3 (one-shot) and K5 (ring): the bits of
    the oracle with the same decay."""
    buckets = [65537, 3]
    T, wd = 5, 1e-2
    X, V = _launch(tmp_path, 2, n, 2, T, buckets, mode, path=path, wd=wd)
    x = np.tile(synth.x0_host(sum(buckets)), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, 2, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     weight_decay=wd)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- NVLS (path 5), group_size = n
def _nvls_or_skip(tmp_path, gpus, n, mode, buckets, T):
    if _TRANSPORT == "loopback":
        pytest.skip("NVLS needs an NVSwitch multicast object across GPUs")
    try:
        return _launch(tmp_path, gpus, n, n, T, buckets, mode, path=5)
    except AssertionError as e:
        if "multicast" in str(e):
            pytest.skip("no NVSwitch multicast on this box")
        raise


@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_nvls_bitexact(tmp_path, mode):
    """NVLS with n = m = 2: the switch adds two values (a + b = b + a), so even the in-switch
    reduction gives the oracle's bits."""
    buckets = [100003, 7, 4096]
    X, V = _nvls_or_skip(tmp_path, 2, 2, mode, buckets, 5)
    x, v = _oracle(2, 2, sum(buckets), 5, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("mode", [0, 1])
def test_four_gpus_nvls(tmp_path, mode):
    """NVLS with n = m = 4 (Ring-SGD's single group): within the north-star tolerance of the
    oracle (the switch's summation order is unspecified) and every worker byte-identical."""
    buckets = [200003, 5]
    X, V = _nvls_or_skip(tmp_path, 4, 4, mode, buckets, 5)
    x, v = _oracle(4, 4, sum(buckets), 5, mode)
    np.testing.assert_allclose(X, x, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(V, v, rtol=1e-5, atol=1e-7)
    assert all(np.array_equal(X[0], X[i]) for i in range(4))


@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_bf16_payload(tmp_path, mode):
    """NEXT-4: the two-shot reduce-scatter in bf16 (SESGD_OPT_PAYLOAD_BF16): the bits of the oracle's
    payload_bf16 reading (R21), over several iterations and ragged buckets."""
    buckets = [100003, 7, 4096]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, mode, path=4, bf16=1)
    x = np.tile(synth.x0_host(sum(buckets)), (2, 1))
    v = np.zeros_like(x)
    oracle.run_local(2, 2, 42, 5, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     payload_bf16=True)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("n,m,mode", [(4, 2, 0), (8, 4, 1), (8, 2, 0)])
def test_two_gpus_bf16_payload_several_workers_per_gpu(tmp_path, n, m, mode):
    """NEXT-4: bf16 payload with n/2 workers per GPU (MULTI kernel): co-resident contributions are
    packed in the contributor's stage, remote ones in the owner's slot, all-local groups round in
    registers -- every fold equals the oracle's payload_bf16 reading (R21) bit for bit."""
    buckets = [100003, 7, 4096]
    X, V = _launch(tmp_path, 2, n, m, 5, buckets, mode, path=4, bf16=1)
    x = np.tile(synth.x0_host(sum(buckets)), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, 5, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     payload_bf16=True)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- K4, value-carried validity
# SESGD_OPT_PROTOCOL = 1: no flags and no sender fence; every receive float is armed with a
# sentinel NaN, the receiver polls the values themselves and re-arms them.  Same bits as the
# oracle (the arithmetic and fold order are K4's).
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_twoshot_value_protocol(tmp_path, mode, fused):
    buckets = [100003, 7, 40000, 4096]
    X, V = _launch(tmp_path, 2, 2, 2, 6, buckets, mode, fused=fused, path=4, protocol=1)
    x, v = _oracle(2, 2, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("lag,grid", [(1, 8), (2, 24), (3, 0), (64, 4)])
def test_two_gpus_value_protocol_pipeline_shapes(tmp_path, lag, grid):
    """many chunks per CTA and every lag: slots are re-armed and reused (call parity) across 5
    iterations, including CTAs whose whole chunk list sits inside one lag"""
    buckets = [250001, 13, 70000]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, grid=grid, lag=lag, path=4, protocol=1)
    x, v = _oracle(2, 2, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("n,m,mode", [(8, 2, 0), (8, 4, 1), (4, 2, 1)])
def test_two_gpus_value_protocol_several_workers_per_gpu(tmp_path, n, m, mode):
    """MULTI: co-resident members through the stage, remote ones through re-armed slots"""
    buckets = [60001, 4097]
    X, V = _launch(tmp_path, 2, n, m, 6, buckets, mode, path=4, protocol=1)
    x, v = _oracle(n, m, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m", [2, 4])
def test_four_gpus_value_protocol(tmp_path, m):
    buckets = [200003, 5000, 1]
    X, V = _launch(tmp_path, 4, 4, m, 5, buckets, path=4, protocol=1)
    x, v = _oracle(4, m, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("gpus", [8, 2])
def test_value_protocol_resnet50_bench_shape(tmp_path, gpus):
    """cfg 2 at full size (n = 8, m = 2, 5 ResNet-50 buckets, T = 100) through protocol 1"""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    buckets = list(RESNET50_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, gpus, 8, 2, 100, buckets, coords=coords, path=4, protocol=1)
    x, v = _oracle(8, 2, sum(buckets), 100, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- K4W: warp-specialised two-shot
# SESGD_OPT_PROTOCOL = 2 (one worker per GPU, one CTA per SM): stream / fold / gather warp groups
# joined only by a shared-memory ring (mbarriers) and by value-carried validity over NVLink.
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("mode", [0, 1])
def test_two_gpus_k4w(tmp_path, mode, fused):
    buckets = [100003, 7, 40000, 4096]
    X, V = _launch(tmp_path, 2, 2, 2, 6, buckets, mode, fused=fused, path=4, protocol=2)
    x, v = _oracle(2, 2, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("grid", [1, 3, 8])
def test_two_gpus_k4w_small_grids(tmp_path, grid):
    """many chunks per CTA: the ring wraps (S waits for R to free entries) and the receive slots
    of both call parities are re-armed and reused over 5 iterations"""
    buckets = [250001, 13, 70000]
    X, V = _launch(tmp_path, 2, 2, 2, 5, buckets, grid=grid, path=4, protocol=2)
    x, v = _oracle(2, 2, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m,mode", [(2, 0), (4, 0), (4, 1)])
def test_four_gpus_k4w(tmp_path, m, mode):
    buckets = [200003, 5000, 1]
    X, V = _launch(tmp_path, 4, 4, m, 5, buckets, mode, path=4, protocol=2)
    x, v = _oracle(4, m, sum(buckets), 5, mode)
    _compare(X, x)
    _compare(V, v)


def test_k4w_resnet50_north_star_shape(tmp_path):
    """the north star's 8-GPU layout: n = 8 workers, one per rank, group_size 2, the five
    ResNet-50 buckets at full size, T = 100, through K4W; sampled coordinates vs the oracle"""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    buckets = list(RESNET50_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, 8, 8, 2, 100, buckets, coords=coords, path=4, protocol=2)
    x, v = _oracle(8, 2, sum(buckets), 100, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("protocol,mode", [(1, 0), (2, 0), (2, 1)])
def test_two_gpus_value_protocols_weight_decay(tmp_path, protocol, mode):
    buckets = [65537, 3]
    T, wd = 5, 1e-2
    X, V = _launch(tmp_path, 2, 2, 2, T, buckets, mode, path=4, wd=wd, protocol=protocol)
    x = np.tile(synth.x0_host(sum(buckets)), (2, 1))
    v = np.zeros_like(x)
    oracle.run_local(2, 2, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     weight_decay=wd)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- stress: 1000 iterations, random shapes
def _stress_cases(k=6, seed=2024):
    """random (ranks, n, m, protocol, grid, lag, release_every, mode): every flag / slot / ring
    reuse path over 1000 iterations (both call parities ~500 times)"""
    rng = np.random.default_rng(seed)
    cases = []
    while len(cases) < k:
        gpus = int(rng.choice([2, 4]))
        n = gpus * int(rng.choice([1, 2]))
        m = int(rng.choice([d for d in (2, 4, 8) if n % d == 0 and d <= n]))
        r = n // gpus
        protocol = int(rng.choice([0, 1, 2] if r == 1 else [0, 1]))
        grid = int(rng.choice([0, 3, 8, 16]))
        lag = int(rng.integers(1, 6))
        rel = int(rng.integers(1, 5))
        mode = int(rng.integers(0, 2))
        cases.append((gpus, n, m, protocol, grid, lag, rel, mode))
    return cases


@pytest.mark.parametrize("gpus,n,m,protocol,grid,lag,rel,mode", _stress_cases())
def test_stress_thousand_iterations_random_shapes(tmp_path, gpus, n, m, protocol, grid, lag, rel, mode):
    buckets = [3001, 17, 4099]
    T = 1000
    X, V = _launch(tmp_path, gpus, n, m, T, buckets, mode, grid=grid, lag=lag, path=4, protocol=protocol,
                   release_every=rel)
    x, v = _oracle(n, m, sum(buckets), T, mode)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- K4W-M: several workers per GPU
# SESGD_OPT_PROTOCOL 2 with r > 1 (p2p_wsm.cu): units = pieces of one slice of one chunk for every
# local worker; all-local groups folded in S, spanning groups through the x_hat ring / NVLink.
@pytest.mark.parametrize("n,m,mode", [(4, 2, 0), (8, 2, 0), (8, 2, 1), (8, 4, 0), (8, 4, 1), (16, 8, 0)])
def test_two_ranks_k4w_multi(tmp_path, n, m, mode):
    buckets = [60001, 4097, 3]
    X, V = _launch(tmp_path, 2, n, m, 6, buckets, mode, path=4, protocol=2)
    x, v = _oracle(n, m, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("grid,fused", [(1, 1), (3, 0), (8, 1)])
def test_two_ranks_k4w_multi_small_grids(tmp_path, grid, fused):
    buckets = [250001, 13, 70000]
    X, V = _launch(tmp_path, 2, 8, 2, 5, buckets, grid=grid, fused=fused, path=4, protocol=2)
    x, v = _oracle(8, 2, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("m", [2, 4])
def test_four_ranks_k4w_multi(tmp_path, m):
    buckets = [200003, 5000, 1]
    X, V = _launch(tmp_path, 4, 8, m, 5, buckets, path=4, protocol=2)
    x, v = _oracle(8, m, sum(buckets), 5, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("gpus", [4, 2])
def test_k4w_multi_resnet50_bench_shape(tmp_path, gpus):
    """cfg 2 at full size through K4W-M: n = 8, m = 2, 2 / 4 workers per rank, T = 100"""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    buckets = list(RESNET50_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, gpus, 8, 2, 100, buckets, coords=coords, path=4, protocol=2)
    x, v = _oracle(8, 2, sum(buckets), 100, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("n,m,mode,fused", [(8, 2, 0, 1), (8, 4, 1, 1), (16, 2, 0, 0)])
def test_k4w_multi_hybrid(tmp_path, n, m, mode, fused):
    """SESGD_OPT_WSM_HYBRID: K6 updates the all-local groups, K4W-M the spanning ones -- same bits"""
    buckets = [60001, 4097, 3]
    X, V = _launch(tmp_path, 2, n, m, 6, buckets, mode, fused=fused, path=4, protocol=2, hybrid=1)
    x, v = _oracle(n, m, sum(buckets), 6, mode)
    _compare(X, x)
    _compare(V, v)


def test_k4w_multi_weight_decay(tmp_path):
    buckets = [65537, 3]
    T, wd = 5, 1e-2
    X, V = _launch(tmp_path, 2, 4, 2, T, buckets, 1, path=4, wd=wd, protocol=2)
    x = np.tile(synth.x0_host(sum(buckets)), (4, 1))
    v = np.zeros_like(x)
    oracle.run_local(4, 2, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=1, weight_decay=wd)
    _compare(X, x)
    _compare(V, v)


# ---------------------------------------------------------------- device-resident iteration state
# SESGD_OPT_DEVICE_ITER: t, its groups (evaluated on the GPU) and the exchange call
# history in device memory.  devit 1: sesgd_begin_iter_device + the gradient fill reading the
# device's t + sync, enqueued per iteration; 2: that iteration captured ONCE as a CUDA graph and
# replayed T times; 3: host iterations, graph replays, host iterations (state host -> device -> host).
@pytest.mark.parametrize("devit", [1, 2, 3])
@pytest.mark.parametrize("gpus,n,m,path", [(2, 2, 2, 4), (4, 8, 2, 4), (2, 8, 4, 4), (4, 4, 2, 3), (4, 4, 4, 3)])
def test_device_iteration_state(tmp_path, devit, gpus, n, m, path):
    """K4W (one worker per rank), K4W-M (several) and the paper's ring K5 (path 3), bit-exact vs
    the oracle over T = 9 iterations (both call parities, several schedules)"""
    buckets = [70001, 4099, 333]
    X, V = _launch(tmp_path, gpus, n, m, 9, buckets, path=path, protocol=2 if path == 4 else -1, devit=devit)
    x, v = _oracle_ring(n, m, buckets, 9, 0) if path == 3 else _oracle(n, m, sum(buckets), 9, 0)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("fused,mode", [(0, 0), (0, 1), (1, 1)])
def test_device_iteration_graph_per_bucket_and_grad(tmp_path, fused, mode):
    """per-bucket launches (per-layer mode) inside the graph, and GRAD mode; t0 > 0 (resume)"""
    buckets = [30001, 7, 4096, 1, 12345]
    X, V = _launch(tmp_path, 2, 4, 2, 7, buckets, mode, t0=11, fused=fused, path=4, protocol=2, devit=2)
    x, v = _oracle(4, 2, sum(buckets), 7, mode, t0=11)
    _compare(X, x)
    _compare(V, v)


def test_device_iteration_resnet50_graph(tmp_path):
    """the north star's one-worker-per-GPU layout at n = 4, the five ResNet-50 buckets at full size,
    T = 30 graph replays, sampled coordinates"""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    buckets = list(RESNET50_BUCKETS)
    coords = _sample(buckets)
    X, V = _launch(tmp_path, 4, 4, 2, 30, buckets, coords=coords, path=4, protocol=2, devit=2)
    x, v = _oracle(4, 2, sum(buckets), 30, 0, coords=coords)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("gpus,n,m,grid,mode", [(2, 2, 2, 3, 0), (2, 8, 2, 0, 1), (4, 8, 4, 8, 0), (4, 4, 2, 0, 1)])
def test_stress_device_iteration_graph(tmp_path, gpus, n, m, grid, mode):
    """500 replays of ONE captured iteration graph (device-resident t, groups and call history;
    K4W / K4W-M, small grids so every CTA walks many chunks and both call parities recycle the
    receive slots hundreds of times), bit-exact with the oracle"""
    buckets = [3001, 17, 4099]
    T = 500
    X, V = _launch(tmp_path, gpus, n, m, T, buckets, mode, grid=grid, path=4, protocol=2, devit=2)
    x, v = _oracle(n, m, sum(buckets), T, mode)
    _compare(X, x)
    _compare(V, v)

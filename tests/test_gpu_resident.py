"""GPU parity of the 1-GPU path (K6, all n workers resident) against the CPU oracle.

Every test drives the C ABI (through SESGDEngine / the ctypes binding), fills the
seeded synthetic inputs on the device (synth/), runs T iterations and compares
element by element with oracle.run on the same inputs.  Bar (BASELINE north star):
<= 1e-5 relative with atol 1e-7 (fp32); the kernels use the oracle's binary32 op
order, so the comparison is additionally asserted bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-7
LR, MU = 0.1, 0.9


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_00433_b200.engine import SESGDEngine
    return SESGDEngine


def _run_gpu(n, m, buckets, T, mode, seed=42, fused=True, unroll=0):
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    eng = SESGDEngine(n, m, buckets, seed=seed, mode=mode, options={C.OPT_RESIDENT_UNROLL: unroll})
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    stream = torch.cuda.current_stream()
    for s in range(eng.r):
        for b, L in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), stream.cuda_stream)
    for t in range(T):
        for s, w in enumerate(eng.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, t, stream.cuda_stream)
        eng.step(t, LR, MU, fused=fused)
    torch.cuda.synchronize()
    eng.poll()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(eng.r)])
    V = np.stack([torch.cat([eng.v(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(eng.r)])
    stats = [eng.stats(b) for b in range(len(buckets))]
    eng.close()
    return X, V, stats


def _run_oracle(n, m, L, T, mode, seed=42, coords=None):
    S = L if coords is None else len(coords)
    x = np.tile(synth.x0_host(S, coords=coords), (n, 1))
    v = np.zeros_like(x)
    oracle.run(n, m, seed, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=mode, coords=coords)
    return x, v


def _compare(got, want):
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    mism = int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
    assert mism == 0, f"{mism} elements differ in bits (within tolerance)"


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_config1_full_parity(mode, fused):
    """BASELINE configs[0]: n=4, group_size=2, 3 odd-sized buckets totalling 2^20, T=8; one
    all-bucket launch per iteration (sesgd_sync_all) or one launch per bucket."""
    from paper_2007_00433_b200.workloads import CONFIG1_BUCKETS
    n, m, T = 4, 2, 8
    X, V, stats = _run_gpu(n, m, CONFIG1_BUCKETS, T, mode, fused=fused)
    x, v = _run_oracle(n, m, sum(CONFIG1_BUCKETS), T, mode)
    _compare(X, x)
    _compare(V, v)
    assert all(s["sync_calls"] == T for s in stats)
    assert sum(s["kernel_launches"] for s in stats) == (T if fused else T * len(CONFIG1_BUCKETS))


@pytest.mark.parametrize("unroll", [2, 4, 8])
def test_resident_unroll_variants(unroll):
    """Every K6 unroll variant (SESGD_OPT_RESIDENT_UNROLL) gives the oracle's bits."""
    buckets = [300007, 5, 40000]
    X, V, _ = _run_gpu(8, 2, buckets, 4, oracle.MODE_PARAM, unroll=unroll)
    x, v = _run_oracle(8, 2, sum(buckets), 4, oracle.MODE_PARAM)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("n,m", [(4, 1), (4, 4), (8, 2), (8, 4), (8, 8), (6, 3), (16, 4), (12, 6)])
@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_group_sizes_and_ragged_tails(n, m, mode):
    """m in {1, n, 2, 4, 8} (templated kernels) and 3, 6 (runtime-m kernel); bucket sizes that
    span several CTAs, ragged tails of 1-3 elements, an empty bucket and a 1-element bucket."""
    buckets = [70001, 0, 1, 4099, 12345]
    T = 5
    X, V, _ = _run_gpu(n, m, buckets, T, mode)
    x, v = _run_oracle(n, m, sum(buckets), T, mode)
    _compare(X, x)
    _compare(V, v)


def test_unaligned_pointers_take_scalar_path():
    """Pointers not 16-byte aligned: the scalar kernel gives the same bits."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    n, m, L, T = 4, 2, 10007, 4
    dev = torch.device("cuda", 0)
    xs = [torch.zeros(L + 1, device=dev) for _ in range(n)]
    vs = [torch.zeros(L + 1, device=dev) for _ in range(n)]
    gs = [torch.zeros(L + 1, device=dev) for _ in range(n)]
    ctx = C.sesgd_init(n, m, 42)
    C.sesgd_attach(ctx, 0, list(range(n)))
    ptr = lambda t: t.data_ptr() + 4  # noqa: E731  (offset by one float: 4-byte aligned only)
    C.sesgd_register_bucket(ctx, 0, L, [ptr(t) for t in xs], [ptr(t) for t in vs], [ptr(t) for t in gs])
    st = torch.cuda.current_stream().cuda_stream
    for i in range(n):
        synth.fill_x0_device(ptr(xs[i]), L, 0, st)
    for t in range(T):
        for i in range(n):
            synth.fill_grad_device(ptr(gs[i]), L, 0, i, t, st)
        C.sesgd_begin_iter(ctx, t)
        C.sesgd_sync_step(ctx, 0, LR, MU, st)
    torch.cuda.synchronize()
    X = np.stack([t[1:].cpu().numpy() for t in xs])
    C.sesgd_destroy(ctx)
    x, _ = _run_oracle(n, m, L, T, oracle.MODE_PARAM)
    _compare(X, x)


def test_random_access_iterations_and_resume():
    """sesgd_begin_iter(t) at arbitrary t (S:152 restart): iterations t0..t0+T-1 equal the
    oracle started at t0."""
    SESGDEngine = _cuda()
    n, m, L, t0, T = 8, 2, 30000, 1000, 3
    eng = SESGDEngine(n, m, [L])
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        synth.fill_x0_device(eng.x(s, 0).data_ptr(), L, 0, st)
    for t in range(t0, t0 + T):
        for s in range(n):
            synth.fill_grad_device(eng.g(s, 0).data_ptr(), L, 0, s, t, st)
        eng.step(t, LR, MU)
    torch.cuda.synchronize()
    X = np.stack([eng.x(s, 0).cpu().numpy() for s in range(n)])
    eng.close()
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, t0=t0)
    _compare(X, x)


def test_resnet50_full_size_sampled():
    """BASELINE configs[1] at full size on one GPU (8 resident workers, group_size 2, the five
    ResNet-50 DDP buckets, 25,557,032 fp32 each) for T=100 iterations, in the launch
    configuration bench.py times; the oracle replays 3000 sampled coordinates (bucket edges,
    ragged tails, random interior) of the same run."""
    from paper_2007_00433_b200.workloads import RESNET50_BUCKETS
    SESGDEngine = _cuda()
    n, m, T = 8, 2, 100
    buckets = list(RESNET50_BUCKETS)
    L = sum(buckets)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    rng = np.random.default_rng(11)
    edges = np.concatenate([[o, o + 1, o + s - 1, o + s - 2] for o, s in zip(offs, buckets)])
    coords = np.unique(np.concatenate([edges, rng.integers(0, L, 3000 - len(edges))])).astype(np.int64)
    eng = SESGDEngine(n, m, buckets)
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st)
    for t in range(T):
        for s in range(n):
            for b, Lb in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), s, t, st)
        eng.step(t, LR, MU)
    torch.cuda.synchronize()
    idx = torch.from_numpy(coords).cuda()
    X = np.stack([eng.x_flat[s][_padded(idx, buckets, eng.offsets)].cpu().numpy() for s in range(n)])
    V = np.stack([eng.v_flat[s][_padded(idx, buckets, eng.offsets)].cpu().numpy() for s in range(n)])
    eng.close()
    x, v = _run_oracle(n, m, L, T, oracle.MODE_PARAM, coords=coords)
    _compare(X, x)
    _compare(V, v)


def _padded(idx, buckets, offsets):
    """map global (unpadded) element indices to the engine's aligned flat layout"""
    starts = torch.tensor(np.concatenate([[0], np.cumsum(buckets)[:-1]]), device=idx.device)
    b = torch.searchsorted(starts, idx, right=True) - 1
    return idx - starts[b] + torch.tensor(offsets, device=idx.device)[b]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_local_sesgd_and_final_global_average(mode, fused):
    """NEXT-2: Local-SESGD with period H = 3 (SESGD_OPT_LOCAL_PERIOD; exchange only when
    (t + 1) % 3 == 0), then Algorithm 1's final global average (K8): the oracle's
    bits after every stage."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    n, m, T, H = 8, 2, 7, 3
    buckets = [30001, 5, 4096]
    L = sum(buckets)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(n, m, buckets, mode=mode, options={C.OPT_LOCAL_PERIOD: H})
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st)
    for t in range(T):
        for s in range(n):
            for b, Lb in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), s, t, st)
        eng.step(t, LR, MU, fused=fused)
    torch.cuda.synchronize()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    V = np.stack([torch.cat([eng.v(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, period=H, mode=mode)
    _compare(X, x)
    _compare(V, v)
    assert sum(eng.stats(b)["kernel_launches"] for b in range(len(buckets))) == (T if fused else T * 3)
    eng.global_average()
    torch.cuda.synchronize()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    eng.close()
    _compare(X, oracle.global_average(x.copy()))


@pytest.mark.parametrize("n,m,period", [(8, 2, 1), (16, 4, 2), (4, 2, 1)])
def test_dimension_exchange_schedule(n, m, period):
    """NEXT-3: Stone's dimension-exchange schedule (SESGD_OPT_SCHEDULE = 1), optionally with a
    local period: the oracle's bits (its own schedule implementation)."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    T, buckets = 6, [20001, 3]
    L = sum(buckets)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(n, m, buckets, options={C.OPT_SCHEDULE: 1, C.OPT_LOCAL_PERIOD: period})
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st)
    for t in range(T):
        for s in range(n):
            for b, Lb in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), s, t, st)
        eng.step(t, LR, MU)
    torch.cuda.synchronize()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    eng.close()
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, period=period,
                     schedule=oracle.SCHED_STONE)
    _compare(X, x)


@pytest.mark.parametrize("pipelined", [True, False])
def test_host_buffer_path(pipelined):
    """The end-to-end host-buffer calls (sesgd_sync_all_host pipelined on copy streams, and
    sesgd_sync_step_host per bucket): pinned host gradients in, updated parameters out, the
    oracle's bits."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200.workloads import CONFIG1_BUCKETS
    n, m, T = 4, 2, 3
    buckets = list(CONFIG1_BUCKETS)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(n, m, buckets)
    st = torch.cuda.current_stream()
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st.cuda_stream)
    g_host = [[torch.empty(Lb).pin_memory() for _ in range(n)] for Lb in buckets]
    x_host = [[torch.empty(Lb).pin_memory() for _ in range(n)] for Lb in buckets]
    for t in range(T):
        for b, Lb in enumerate(buckets):
            for s in range(n):
                g_host[b][s].copy_(torch.from_numpy(synth.grad_host(s, t, Lb, e0=int(offs[b]))))
        eng.step_host(t, LR, MU, g_host, x_host, pipelined=pipelined)
        torch.cuda.synchronize()
    X = np.stack([np.concatenate([x_host[b][s].numpy() for b in range(len(buckets))]) for s in range(n)])
    eng.close()
    x, _ = _run_oracle(n, m, sum(buckets), T, oracle.MODE_PARAM)
    _compare(X, x)


def test_consensus_metric():
    """NEXT-4: the device consistency metric (K9, binary64) equals the oracle's on the state after
    10 SESGD iterations, and is exactly 0 right after the final global average."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200.workloads import CONFIG1_BUCKETS
    n, m, T = 8, 2, 10
    buckets = list(CONFIG1_BUCKETS)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(n, m, buckets)
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st)
    for t in range(T):
        for s in range(n):
            for b, Lb in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), s, t, st)
        eng.step(t, LR, MU)
    ss, mx = eng.consensus()
    x, _ = _run_oracle(n, m, sum(buckets), T, oracle.MODE_PARAM)
    oss, omx = oracle.consensus(x)
    assert ss > 0 and abs(ss - oss) <= 1e-9 * oss
    assert abs(mx - omx) <= 1e-12 * omx
    eng.global_average()
    assert eng.consensus() == (0.0, 0.0)
    eng.close()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
@pytest.mark.parametrize("n,m", [(8, 2), (6, 3), (4, 1)])
def test_weight_decay(n, m, mode, fused):
    """NEXT-4: weight decay folded into the update (sesgd_set_weight_decay; the WD-compiled K6
    kernels, templated and runtime m), the oracle's bits."""
    SESGDEngine = _cuda()
    T, buckets, wd = 5, [30001, 7], 1e-2
    L = sum(buckets)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(n, m, buckets, mode=mode, weight_decay=wd)
    st = torch.cuda.current_stream().cuda_stream
    for s in range(n):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), st)
    for t in range(T):
        for s in range(n):
            for b, Lb in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), s, t, st)
        eng.step(t, LR, MU, fused=fused)
    torch.cuda.synchronize()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    V = np.stack([torch.cat([eng.v(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(n)])
    eng.close()
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, 42, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, period=1, mode=mode,
                     weight_decay=wd)
    _compare(X, x)
    _compare(V, v)


@pytest.mark.parametrize("n,m,schedule", [(8, 2, 0), (16, 4, 0), (6, 3, 0), (8, 2, 1), (16, 4, 1)])
def test_pair_counts_on_device(n, m, schedule):
    """NEXT-4: the schedule evaluated on the device (K10) counts the same co-memberships as the
    oracle's schedule over 3000 iterations (integers: exact)."""
    _cuda()
    from paper_2007_00433_b200 import sesgd as C
    ctx = C.sesgd_init(n, m, 42)
    try:
        if schedule:
            C.sesgd_set_option(ctx, C.OPT_SCHEDULE, 1)
        C.sesgd_attach(ctx, 0, list(range(n)))
        counts = torch.zeros(n * n, dtype=torch.int64, device="cuda")
        t0, T = 17, 3000
        C.sesgd_pair_counts(ctx, t0, T, counts.data_ptr(), torch.cuda.current_stream().cuda_stream)
        got = counts.cpu().numpy().reshape(n, n)
    finally:
        C.sesgd_destroy(ctx)
    want = np.zeros((n, n), np.int64)
    for t in range(t0, t0 + T):
        gof = oracle.groups_stone(t, n, m)[1] if schedule else oracle.groups(42, t, n, m)[2]
        for i in range(n):
            for j in range(i + 1, n):
                want[i, j] += int(gof[i] == gof[j])
    assert np.array_equal(got, want)


def test_pair_split_probability_on_device():
    """P5 / P:498 at scale: over 4 M iterations of the random schedule the pair-split frequency of
    every pair matches n (k - 1) / (k (n - 1)) within 5 sigma (n = 16, k = 4: 0.8)."""
    _cuda()
    from paper_2007_00433_b200 import sesgd as C
    n, m, T = 16, 4, 4_000_000
    ctx = C.sesgd_init(n, m, 42)
    try:
        C.sesgd_attach(ctx, 0, list(range(n)))
        counts = torch.zeros(n * n, dtype=torch.int64, device="cuda")
        C.sesgd_pair_counts(ctx, 0, T, counts.data_ptr(), torch.cuda.current_stream().cuda_stream)
        together = counts.cpu().numpy().reshape(n, n)[np.triu_indices(n, 1)]
    finally:
        C.sesgd_destroy(ctx)
    k = n // m
    p_split = n * (k - 1) / (k * (n - 1))
    split = T - together
    sigma = np.sqrt(T * p_split * (1 - p_split))
    assert abs(p_split - 0.8) < 1e-15
    assert np.all(np.abs(split - T * p_split) < 5 * sigma)


def test_bf16_payload_rejected_on_resident_path():
    """R21 rounds what crosses NVLink (K4); K6 keeps every contribution fp32, so asking for the
    bf16 payload with every worker resident is refused rather than silently ignored."""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    eng = SESGDEngine(4, 2, [1000], seed=42, options={C.OPT_PAYLOAD_BF16: 1})
    eng.begin_iter(0)
    with pytest.raises(C.SesgdError) as ei:
        eng.sync_all(LR, MU)
    assert ei.value.code == C.ENOTSUP
    with pytest.raises(C.SesgdError) as ei:
        eng.sync_step(0, LR, MU)
    assert ei.value.code == C.ENOTSUP
    eng.close()


# ---------------------------------------------------------------- device-resident iteration state
@pytest.mark.parametrize("n,m,mode,fused", [(8, 2, 0, True), (8, 2, 1, True), (8, 4, 0, False), (12, 3, 0, True),
                                            (16, 16, 0, True)])
def test_device_iteration_graph_resident(n, m, mode, fused):
    """SESGD_OPT_DEVICE_ITER on the 1-GPU path (K6): ONE captured CUDA graph of [begin_iter_device
    (next t, groups evaluated on the GPU), gradient fill reading the device's t, sync] replayed for
    T iterations is bit-exact with the oracle; switching the option off hands t back to the host,
    which continues with two host iterations"""
    SESGDEngine = _cuda()
    from paper_2007_00433_b200 import sesgd as C
    buckets = [699_051, 262_147, 87_378]
    T = 7
    eng = SESGDEngine(n, m, buckets, seed=42, mode=mode)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    st = torch.cuda.current_stream().cuda_stream
    for s in range(eng.r):
        for b, L in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), st)
    eng.set_device_iter(True)
    with pytest.raises(C.SesgdError):  # the host may not move t while the device owns it
        eng.begin_iter(0)

    def produce(e, s):
        tp = e.t_device_ptr()
        for slot, w in enumerate(e.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_grad_device_at(e.g(slot, b).data_ptr(), L, int(offs[b]), w, tp, s.cuda_stream)

    g = eng.capture_iteration(LR, MU, produce, fused)
    for _ in range(T):
        eng.replay_iteration(g)
    torch.cuda.synchronize()
    state = C.sesgd_device_iter_read(eng.ctx, n, m)
    assert state["t"] == T - 1  # from "no iteration" (-1), one step per replay
    assert sorted(state["canon"]) == list(range(n))
    assert state["canon"] == [int(w) for w in eng.groups(T - 1)[0]]
    eng.set_device_iter(False)
    for t in (T, T + 1):  # the host continues from the device's t
        for s, w in enumerate(eng.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, t, st)
        eng.step(t, LR, MU, fused=fused)
    torch.cuda.synchronize()
    eng.poll()
    X = np.stack([torch.cat([eng.x(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(eng.r)])
    V = np.stack([torch.cat([eng.v(s, b) for b in range(len(buckets))]).cpu().numpy() for s in range(eng.r)])
    eng.close()
    x, v = _run_oracle(n, m, sum(buckets), T + 2, mode)
    _compare(X, x)
    _compare(V, v)


def test_device_iteration_schedule_matches_host():
    """the device's groups for t (sesgd_begin_iter_device, K6 reads them) equal sesgd_groups(t):
    one device iteration at a time, with lr = 0 and distinct x per worker, the K6 update is the
    group mean -- compare it with the host schedule's group means over 40 random t"""
    SESGDEngine = _cuda()
    n, m = 16, 4
    eng = SESGDEngine(n, m, [1024], seed=7)
    eng.set_device_iter(True)
    rng = np.random.default_rng(3)
    for t in rng.integers(0, 2**40, 40):
        x0 = rng.standard_normal((n, 1024)).astype(np.float32)
        for s in range(n):
            eng.x(s, 0).copy_(torch.from_numpy(x0[s]))
            eng.g(s, 0).zero_()
            eng.v(s, 0).zero_()
        eng.begin_iter_device(int(t))
        eng.sync_all(0.0, 0.0)
        torch.cuda.synchronize()
        perm, _ = eng.groups(int(t))
        got = np.stack([eng.x(s, 0).cpu().numpy() for s in range(n)])
        for j in range(n // m):
            G = sorted(perm[j * m:(j + 1) * m])
            acc = x0[G[0]].copy()
            for w in G[1:]:
                acc = (acc + x0[w]).astype(np.float32)
            for w in G:
                assert np.array_equal(got[w], (acc * np.float32(0.25)).astype(np.float32)), (t, G)
    eng.close()

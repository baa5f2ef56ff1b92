"""Pins for the CPU oracle (oracle/): checks against what the paper and the
mathematics fix, never against the oracle's own formulas retyped.

P:n = PAPER.md line n, S:n = SPEC.md line n; P1..P15 = DESIGN.md "Oracle pins".
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

SEED = 42


# ---------------------------------------------------------------- P1: PRNG
def test_splitmix64_golden(golden_dir):
    """P1: splitmix64 golden values (survey scratch script)."""
    rows = []
    for line in open(os.path.join(golden_dir, "splitmix64.txt")):
        line = line.split("#")[0].strip()
        if line:
            s, i, v = line.split()
            rows.append((int(s), int(i), int(v, 16)))
    assert len(rows) == 5
    for seed in {r[0] for r in rows}:
        want = sorted((i, v) for s, i, v in rows if s == seed)
        rng = oracle.Rng64(seed)
        got = [rng.next() for _ in range(len(want))]
        assert got == [v for _, v in want]


def test_bounded_special_cases():
    """R5: bound 1 always 0; bound 0 is an error; power-of-two bounds take every draw."""
    rng = oracle.Rng64(7)
    assert all(rng.bounded(1) == 0 for _ in range(100))
    with pytest.raises(oracle.OracleError):
        rng.bounded(0)
    # bound = 2^k: 2^64 mod 2^k = 0, no rejection -> equals the raw draw's low bits
    a, b = oracle.Rng64(99), oracle.Rng64(99)
    for _ in range(200):
        assert a.bounded(8) == b.next() % 8


def test_bounded_uniform_dice():
    """bound 6, 600000 draws, each face within 5 sigma of 100000."""
    rng = oracle.Rng64(12345)
    counts = np.zeros(6, np.int64)
    for _ in range(600000):
        counts[rng.bounded(6)] += 1
    sigma = math.sqrt(600000 * (1 / 6) * (5 / 6))
    assert np.all(np.abs(counts - 100000) < 5 * sigma), counts


def test_bounded_rejects_top_range():
    """R5: with bound 3, words >= 2^64 - (2^64 mod 3) are rejected, not folded.

    Brute force: simulate the rejection rule with Python big ints on the raw stream."""
    rem = (2 ** 64) % 3
    raw = oracle.Rng64(5)
    rng = oracle.Rng64(5)
    for _ in range(2000):
        got = rng.bounded(3)
        while True:
            w = raw.next()
            if w < 2 ** 64 - rem:
                break
        assert got == w % 3


# ------------------------------------------------------------ schedule pins
def _load_schedules(golden_dir):
    out = []
    for line in open(os.path.join(golden_dir, "schedules_seed42.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        head, groups, raw = [s.strip() for s in line.split(" | ")]
        n, m, t = map(int, head.split())
        gs = [tuple(int(a) for a in g.split(",")) for g in groups.split("|")]
        rawp = None if raw.strip() == "-" else [int(a) for a in raw.split(",")]
        out.append((n, m, t, gs, rawp))
    return out


def test_schedule_golden(golden_dir):
    """P-golden: canonical groups (and raw slots) from an independent script (SURVEY.md:442-452)."""
    rows = _load_schedules(golden_dir)
    assert len(rows) == 16
    for n, m, t, gs, rawp in rows:
        raw, canon, gof = oracle.groups(SEED, t, n, m)
        assert oracle.canonical_groups(SEED, t, n, m) == gs, (n, m, t)
        if rawp is not None:
            assert list(raw) == rawp


def test_schedule_trivial_sizes():
    """P2: m=1 -> singletons, m=n -> one group."""
    for n in (1, 2, 4, 16):
        for t in range(5):
            assert oracle.canonical_groups(SEED, t, n, 1) == [(i,) for i in range(n)]
            assert oracle.canonical_groups(SEED, t, n, n) == [tuple(range(n))]


def test_schedule_errors():
    """R13 / S:129: m must divide n; 1 <= m <= n; t >= 0."""
    with pytest.raises(oracle.OracleError) as e:
        oracle.groups(SEED, 0, 6, 4)
    assert e.value.code == oracle.ENOTDIV
    for bad in [(0, 1), (4, 0), (4, 5)]:
        with pytest.raises(oracle.OracleError):
            oracle.groups(SEED, 0, *bad)
    with pytest.raises(oracle.OracleError):
        oracle.groups(SEED, -1, 4, 2)


def test_schedule_partition_property():
    """P3: every G_t is a partition into n/m groups of size m in canonical form."""
    rng = np.random.default_rng(0)
    for _ in range(400):
        n = int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 32, 64]))
        divs = [d for d in range(1, n + 1) if n % d == 0]
        m = int(rng.choice(divs))
        seed = int(rng.integers(0, 2 ** 63))
        t = int(rng.integers(0, 10 ** 9))
        raw, canon, gof = oracle.groups(seed, t, n, m)
        assert sorted(raw.tolist()) == list(range(n))
        assert sorted(canon.tolist()) == list(range(n))
        k = n // m
        firsts = []
        for j in range(k):
            G = canon[j * m:(j + 1) * m].tolist()
            assert G == sorted(G)
            assert all(gof[a] == j for a in G)
            firsts.append(G[0])
            # the group is exactly one contiguous slice of the raw permutation
            assert any(sorted(raw[s * m:(s + 1) * m].tolist()) == G for s in range(k))
        assert firsts == sorted(firsts)


def test_schedule_determinism_and_random_access():
    """pure function of (seed, t, n, m); any t can be produced directly."""
    a = [oracle.canonical_groups(SEED, t, 16, 4) for t in range(50)]
    b = [oracle.canonical_groups(SEED, t, 16, 4) for t in reversed(range(50))][::-1]
    assert a == b
    assert oracle.canonical_groups(SEED, 10 ** 12, 16, 4) == oracle.canonical_groups(SEED, 10 ** 12, 16, 4)
    assert oracle.canonical_groups(1, 0, 16, 4) != oracle.canonical_groups(2, 0, 16, 4) or \
        oracle.canonical_groups(1, 1, 16, 4) != oracle.canonical_groups(2, 1, 16, 4)


def _all_equal_partitions(n, m):
    """Brute-force enumeration of all partitions of range(n) into blocks of size m."""
    def rec(rest):
        if not rest:
            yield ()
            return
        first = rest[0]
        for others in itertools.combinations(rest[1:], m - 1):
            blk = (first,) + others
            remaining = [a for a in rest if a not in blk]
            for tail in rec(remaining):
                yield (blk,) + tail
    return [list(p) for p in rec(list(range(n)))]


def test_n4_bruteforce_partitions_uniform():
    """P4: n=4, m=2 -> the 3 partitions enumerated by hand, {01|23, 02|13, 03|12},
    each with frequency 1/3 (uniform partition) within 5 sigma over 1e5 t."""
    hand = [[(0, 1), (2, 3)], [(0, 2), (1, 3)], [(0, 3), (1, 2)]]
    assert sorted(_all_equal_partitions(4, 2)) == sorted(hand)
    T = 100000
    counts = {tuple(p): 0 for p in hand}
    for t in range(T):
        counts[tuple(oracle.canonical_groups(SEED, t, 4, 2))] += 1
    assert sum(counts.values()) == T
    sigma = math.sqrt(T * (1 / 3) * (2 / 3))
    for c in counts.values():
        assert abs(c - T / 3) < 5 * sigma, counts


@pytest.mark.parametrize("n,m", [(6, 2), (6, 3)])
def test_small_n_partitions_uniform(n, m):
    """P4 generalised: every equal partition (brute-force enumerated) is equally likely
    (chi-square, p > 1e-4), as the appendix probability requires."""
    parts = _all_equal_partitions(n, m)
    idx = {tuple(p): i for i, p in enumerate(parts)}
    T = 60000
    counts = np.zeros(len(parts))
    for t in range(T):
        counts[idx[tuple(oracle.canonical_groups(7, t, n, m))]] += 1
    exp = T / len(parts)
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    from scipy.stats import chi2 as chi2d
    assert chi2d.sf(chi2, len(parts) - 1) > 1e-4, (chi2, counts)


@pytest.mark.parametrize("n,k", [(4, 2), (16, 4), (8, 4), (8, 2), (16, 2)])
def test_pair_split_probability(n, k):
    """P5: Pr[workers 0 and 1 in different groups] = n(k-1)/(k(n-1)) (appendix;
    S:144: 2/3 at n=4,k=2; 0.8 at n=16,k=4), Monte Carlo within 5 sigma."""
    m = n // k
    p = n * (k - 1) / (k * (n - 1))
    if (n, k) == (4, 2):
        assert abs(p - 2 / 3) < 1e-15
    if (n, k) == (16, 4):
        assert abs(p - 0.8) < 1e-15
    T = 40000
    split = 0
    for t in range(T):
        _, _, gof = oracle.groups(SEED, t, n, m)
        split += int(gof[0] != gof[1])
    sigma = math.sqrt(T * p * (1 - p))
    assert abs(split - T * p) < 5 * sigma, (split / T, p)


# -------------------------------------------------------- update-rule pins
def _W(n, m, t, seed=SEED):
    """Averaging matrix of iteration t: W[i][j] = 1/m iff i, j share a group (Eq. 6, k/n = 1/m)."""
    _, _, gof = oracle.groups(seed, t, n, m)
    return (gof[:, None] == gof[None, :]).astype(np.float64) / m


def test_averaging_matrix_doubly_stochastic():
    """P6: W_t symmetric, doubly stochastic, idempotent; and the oracle step with
    lr=0, mu=0 on distinct x applies exactly W_t (brute-force dense form)."""
    rng = np.random.default_rng(1)
    for n, m in [(4, 2), (8, 2), (8, 4), (16, 4), (6, 3)]:
        for t in range(10):
            W = _W(n, m, t)
            assert np.array_equal(W, W.T)
            assert np.allclose(W.sum(0), 1) and np.allclose(W.sum(1), 1)
            assert np.allclose(W @ W, W)
            X = rng.standard_normal((n, 7))
            x = X.copy()
            v = np.zeros_like(x)
            _, canon, _ = oracle.groups(SEED, t, n, m)
            oracle.step(n, m, canon, x, v, np.zeros_like(x), 0.0, 0.0)
            np.testing.assert_allclose(x, W @ X, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
@pytest.mark.parametrize("n,m", [(4, 2), (8, 4), (6, 3)])
def test_dense_matrix_form_with_momentum(n, m, mode):
    """P12 with lr, momentum != 0: the group-loop oracle equals Algorithm 1 written as dense
    n x n products over T iterations, distinct x_0 and prior momentum.
    PARAM (Eq. 6, R8): V <- mu V + G ; X <- W_t (X - lr V)   (momentum stays local).
    GRAD  (Eq. 5, R8): V <- mu V + W_t G ; X <- X - lr V."""
    rng = np.random.default_rng(n * 10 + m + mode)
    L, lr, mu = 5, 0.1, 0.9
    X = rng.standard_normal((n, L))
    V = rng.standard_normal((n, L))
    x, v = X.copy(), V.copy()
    for t in range(12):
        G = rng.standard_normal((n, L))
        W = _W(n, m, t)
        if mode == oracle.MODE_PARAM:
            V = mu * V + G
            X = W @ (X - lr * V)
        else:
            V = mu * V + W @ G
            X = X - lr * V
        _, canon, _ = oracle.groups(SEED, t, n, m)
        oracle.step(n, m, canon, x, v, G.copy(), lr, mu, mode)
        np.testing.assert_allclose(v, V, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(x, X, rtol=1e-12, atol=1e-13)


def test_hand_step(golden_dir):
    """Hand-executed single step at n=4 (Eq. 6 and Eq. 5 variants), exact dyadic values."""
    d = json.load(open(os.path.join(golden_dir, "hand_step_n4.json")))
    n, m = d["n"], d["m"]
    _, canon, _ = oracle.groups(d["seed"], d["t"], n, m)
    for dt in (np.float32, np.float64):
        for mode, key in [(oracle.MODE_PARAM, "param_x1"), (oracle.MODE_GRAD, "grad_x1")]:
            x = np.array(d["x0"], dt)
            v = np.zeros_like(x)
            oracle.step(n, m, canon, x, v, np.array(d["g"], dt), d["lr"], d["mu"], mode)
            assert np.array_equal(x, np.array(d[key], dt)), (dt, key, x)
        pv = d["param_x1_with_prior_v"]
        for mode, key in [(oracle.MODE_PARAM, "x1"), (oracle.MODE_GRAD, "grad_x1")]:
            x = np.array(d["x0"], dt)
            v = np.array(pv["v0"], dt)
            oracle.step(n, m, canon, x, v, np.array(d["g"], dt), d["lr"], pv["mu"], mode)
            assert np.array_equal(x, np.array(pv[key], dt)), (dt, key, x)


def _synthetic_run(n, m, T, L, mode, dtype, lr=0.1, mu=0.9, seed=SEED, coords=None):
    x = np.tile(synth.x0_host(L, coords=coords).astype(dtype), (n, 1))
    v = np.zeros_like(x)
    oracle.run(n, m, seed, T, x, v, s_g=synth.SEED_G, lr=lr, mu=mu, mode=mode, coords=coords)
    return x, v


def _grads(n, t, L, dtype=np.float64):
    return np.stack([synth.grad_host(i, t, L) for i in range(n)]).astype(dtype)


def _torch_sgd_trajectory(x0, grads_per_t, lr, mu, dtype=torch.float64):
    """Textbook momentum SGD via torch.optim.SGD (library routine): v <- mu v + g, x <- x - lr v."""
    p = torch.nn.Parameter(torch.tensor(x0, dtype=dtype))
    opt = torch.optim.SGD([p], lr=lr, momentum=mu, dampening=0.0, nesterov=False, weight_decay=0.0)
    for g in grads_per_t:
        p.grad = torch.tensor(g, dtype=dtype)
        opt.step()
    return p.detach().numpy()


@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
@pytest.mark.parametrize("n,m", [(4, 2), (8, 4), (8, 2), (6, 3)])
def test_sum_preservation_and_mean_trajectory(n, m, mode):
    """P7 + P8: the worker mean xbar_t follows single-worker momentum SGD on the mean
    gradient gbar_t (torch.optim.SGD), for any schedule, both modes (fp64)."""
    T, L, lr, mu = 12, 33, 0.1, 0.9
    x0 = synth.x0_host(L).astype(np.float64)
    x = np.tile(x0, (n, 1))
    v = np.zeros_like(x)
    gbars = []
    for t in range(T):
        g = _grads(n, t, L)
        gbars.append(g.mean(0))
        _, canon, _ = oracle.groups(SEED, t, n, m)
        xh_sum = (x - lr * (mu * v + g)).sum(0)  # sum of locally-stepped params (PARAM)
        oracle.step(n, m, canon, x, v, g, lr, mu, mode)
        if mode == oracle.MODE_PARAM:
            np.testing.assert_allclose(x.sum(0), xh_sum, rtol=0, atol=1e-13)
    ref = _torch_sgd_trajectory(x0, gbars, lr, mu)
    np.testing.assert_allclose(x.mean(0), ref, rtol=0, atol=1e-13)


def test_group_equals_n_is_ring_sgd():
    """P9: m=n -> every worker equals Ring-SGD (Eq. 4) with momentum, i.e.
    torch.optim.SGD on the global mean gradient; all workers byte-identical (P11)."""
    n, T, L, lr, mu = 8, 15, 41, 0.1, 0.9
    x0 = synth.x0_host(L).astype(np.float64)
    for mode in (oracle.MODE_PARAM, oracle.MODE_GRAD):
        x = np.tile(x0, (n, 1))
        v = np.zeros_like(x)
        gbars = []
        for t in range(T):
            g = _grads(n, t, L)
            gbars.append(g.mean(0))
            _, canon, _ = oracle.groups(SEED, t, n, n)
            oracle.step(n, n, canon, x, v, g, lr, mu, mode)
            assert all(np.array_equal(x[0], x[i]) for i in range(n))
        np.testing.assert_allclose(x[0], _torch_sgd_trajectory(x0, gbars, lr, mu), rtol=0, atol=1e-13)


def test_group_size_one_is_local_sgd():
    """P10: m=1 -> each worker is independent momentum SGD (torch.optim.SGD), both modes."""
    n, T, L, lr, mu = 4, 10, 29, 0.1, 0.9
    x0 = synth.x0_host(L).astype(np.float64)
    for mode in (oracle.MODE_PARAM, oracle.MODE_GRAD):
        x = np.tile(x0, (n, 1))
        v = np.zeros_like(x)
        per_worker = [[] for _ in range(n)]
        for t in range(T):
            g = _grads(n, t, L)
            for i in range(n):
                per_worker[i].append(g[i])
            _, canon, _ = oracle.groups(SEED, t, n, 1)
            oracle.step(n, 1, canon, x, v, g, lr, mu, mode)
        for i in range(n):
            np.testing.assert_allclose(x[i], _torch_sgd_trajectory(x0, per_worker[i], lr, mu),
                                       rtol=0, atol=1e-14)


def test_group_size_one_f32_matches_torch_sgd_f32():
    """P10 in binary32: with m=1 the f32 oracle equals torch.optim.SGD float32 within 1 ulp-level
    tolerance (torch's CPU kernel may contract to FMA, so not asserted bit-exact)."""
    n, T, L, lr, mu = 2, 20, 1000, 0.1, 0.9
    x0 = synth.x0_host(L)
    x = np.tile(x0, (n, 1))
    v = np.zeros_like(x)
    gs = []
    for t in range(T):
        g = _grads(n, t, L, np.float32)
        gs.append(g[0])
        _, canon, _ = oracle.groups(SEED, t, n, 1)
        oracle.step(n, 1, canon, x, v, g, lr, mu)
    ref = _torch_sgd_trajectory(x0, gs, lr, mu, dtype=torch.float32)
    np.testing.assert_allclose(x[0], ref, rtol=1e-6, atol=1e-8)


def test_lr_zero_products_of_W():
    """P14: lr=0 with per-worker distinct x_0: X_T = W_{T-1} ... W_0 X_0 (both modes)."""
    n, m, T, L = 8, 2, 9, 5
    rng = np.random.default_rng(3)
    X0 = rng.standard_normal((n, L))
    x = X0.copy()
    v = np.zeros_like(x)
    P = np.eye(n)
    for t in range(T):
        _, canon, _ = oracle.groups(SEED, t, n, m)
        oracle.step(n, m, canon, x, v, _grads(n, t, L), 0.0, 0.9, oracle.MODE_PARAM)
        P = _W(n, m, t) @ P
    np.testing.assert_allclose(x, P @ X0, rtol=1e-13, atol=1e-14)


def test_gradient_correction_reduces_divergence():
    """P13 (Eq. 5 vs Eq. 6): averaging gradients in shuffled groups lets
    workers drift apart; averaging locally-stepped parameters keeps them together."""
    n, m, T, L = 4, 2, 50, 4096
    div = {}
    for mode in (oracle.MODE_PARAM, oracle.MODE_GRAD):
        x, _ = _synthetic_run(n, m, T, L, mode, np.float64)
        div[mode] = max(np.abs(x[i] - x[j]).max() for i in range(n) for j in range(n))
    assert div[oracle.MODE_GRAD] > 3 * div[oracle.MODE_PARAM], div


def test_f32_oracle_within_rounding_of_f64():
    """The binary32 oracle stays within a derived rounding bound of the binary64 one:
    per iteration each coordinate sees <= (m + 4) roundings of magnitude <= 2^-24 |.|,
    intermediates |x| <= 0.25, |v| <= 0.2, so |err| <= T * (m + 4) * 2^-24 * 0.25 * 2."""
    n, m, T, L = 8, 4, 30, 2000
    x32, v32 = _synthetic_run(n, m, T, L, oracle.MODE_PARAM, np.float32)
    x64, v64 = _synthetic_run(n, m, T, L, oracle.MODE_PARAM, np.float64)
    bound = T * (m + 4) * 2.0 ** -24 * 0.25 * 2
    assert np.abs(x32 - x64).max() < bound
    assert np.abs(x32 - x64).max() > 0  # the f32 path really is binary32


def test_run_equals_steps_and_coordinate_subsets():
    """run() with coordinate subsets replays exactly the columns of a full run
    (coordinates are independent: the update is elementwise)."""
    n, m, T, L = 4, 2, 6, 300
    xf, vf = _synthetic_run(n, m, T, L, oracle.MODE_PARAM, np.float32)
    coords = np.array([0, 7, 123, 299, 150], np.int64)
    xs, vs = _synthetic_run(n, m, T, len(coords), oracle.MODE_PARAM, np.float32, coords=coords)
    assert np.array_equal(xs, xf[:, coords]) and np.array_equal(vs, vf[:, coords])
    # step-by-step drive gives the identical bits
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    for t in range(T):
        _, canon, _ = oracle.groups(SEED, t, n, m)
        oracle.step(n, m, canon, x, v, _grads(n, t, L, np.float32), 0.1, 0.9)
    assert np.array_equal(x, xf)


def test_param_mode_group_members_identical():
    """P11: after every exchange all members of a group hold byte-identical x."""
    n, m, L = 8, 4, 100
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    for t in range(5):
        _, canon, _ = oracle.groups(SEED, t, n, m)
        oracle.step(n, m, canon, x, v, _grads(n, t, L, np.float32), 0.1, 0.9)
        for j in range(n // m):
            G = canon[j * m:(j + 1) * m]
            assert all(np.array_equal(x[G[0]], x[a]) for a in G)


# ------------------------------------------------------------ latency model
def test_latency_worked_examples(golden_dir):
    """P15: worked numbers printed in the paper / SPEC (tests/golden/worked_examples.json)."""
    d = json.load(open(os.path.join(golden_dir, "worked_examples.json")))
    assert oracle.latency(3, 3, 0, 1, 0)["ring_handshakes"] == d["ring_handshakes_m3"]["value"]
    assert 50 * oracle.latency(16, 4, 0, 1, 0)["ring_handshakes"] == d["ring_handshakes_50_layers_n16"]["value"]
    assert 50 * oracle.latency(16, 4, 0, 1, 0)["sesgd_handshakes"] == d["sesgd_handshakes_50_layers_n16_k4"]["value"]
    e = d["eq2_example"]
    r = oracle.latency(e["n"], e["n"], e["G"], e["nu"], e["tau"])
    assert abs(r["ring_s"] - e["value_s"]) < 5e-5
    # pure-latency limit (G -> 0) at n=16, k=4 (m=4): ratio 30/6 = 5
    r = oracle.latency(16, 4, 0.0, 1e9, 5e-3)
    assert r["ratio"] == d["latency_limit_ratio_n16_k4"]["value"]


def test_latency_special_cases():
    """S:498 / S:508: m=1 -> 0 s, 0 handshakes; m=n -> SESGD equals ring; tau=0 -> 2G(m-1)/(m nu);
    bandwidth term approaches 2G/nu (Eq. 2 approximation)."""
    r = oracle.latency(8, 1, 1e6, 1e9, 1e-3)
    assert r["sesgd_s"] == 0 and r["sesgd_handshakes"] == 0 and r["ratio"] == math.inf
    r = oracle.latency(8, 8, 1e6, 1e9, 1e-3)
    assert r["ratio"] == 1.0 and r["ring_s"] == r["sesgd_s"]
    r = oracle.latency(1, 1, 1e6, 1e9, 1e-3)
    assert r["ring_s"] == 0 and r["ratio"] == 1.0
    r = oracle.latency(1024, 1024, 1e6, 1e9, 0.0)
    assert abs(r["ring_s"] - 2e6 / 1e9) / (2e6 / 1e9) < 1e-2
    for bad in [(4, 3, 1, 1, 0), (4, 2, -1, 1, 0), (4, 2, 1, 0, 0), (4, 2, 1, 1, -1), (4, 8, 1, 1, 0)]:
        with pytest.raises(oracle.OracleError):
            oracle.latency(*bad)
    # monotone in tau
    rs = [oracle.latency(16, 4, 1e5, 1e9, tau)["ratio"] for tau in (0, 1e-6, 1e-4, 1e-2)]
    assert rs == sorted(rs)


# ------------------------------------------------------ ring-order group mean
def test_slice_bounds_worked_example():
    """SPEC collectives.slice_bounds: L=37, m=4 -> [0,9),[9,18),[18,27),[27,37);
    L=10, m=2 -> [0,5),[5,10); L=3, m=4 -> sizes {0,1,1,1} (empty slice allowed)."""
    def slices(L, m):
        out = [[] for _ in range(m)]
        for e in range(L):
            out[oracle.slice_of(L, m, e)].append(e)
        return out
    s = slices(37, 4)
    assert [(x[0], x[-1] + 1) for x in s] == [(0, 9), (9, 18), (18, 27), (27, 37)]
    s = slices(10, 2)
    assert [(x[0], x[-1] + 1) for x in s] == [(0, 5), (5, 10)]
    assert sorted(len(x) for x in slices(3, 4)) == [0, 1, 1, 1]


def test_ring_mean_worked_example():
    """S:267 ([PAPER] handshake count, TRIVIAL mean): m=3, inputs [1,1],[2,2],[3,3] -> every
    member gets [2,2].  As a step with lr=1, mu=0, x=0 the payload is -g."""
    canon = np.array([0, 1, 2], np.int32)
    x = np.zeros((3, 2), np.float32)
    v = np.zeros_like(x)
    g = -np.array([[1, 1], [2, 2], [3, 3]], np.float32)
    oracle.step_ring(3, 3, canon, x, v, g, 1.0, 0.0)
    assert np.array_equal(x, np.full((3, 2), 2.0, np.float32))


def test_ring_order_starts_each_slice_at_the_next_member():
    """"slice s accumulated in ring order starting from member (s+1) mod m".  m = 3,
    L = 3 (slice s = element s), payloads chosen so that the summation order decides the binary32
    result: for slice s the members' values are 2^24 at s+1, -2^24 at s+2 and 1 at s.  Starting at
    s+1: (2^24 + -2^24) + 1 = 1, mean fl(1/3).  Starting at s (the other plausible reading):
    (1 + 2^24) rounds to 2^24, + -2^24 = 0.  Hand-computed, not re-derived from the oracle."""
    big = np.float32(2.0 ** 24)
    x = np.zeros((3, 3), np.float32)
    for s in range(3):
        x[(s + 1) % 3, s], x[(s + 2) % 3, s], x[s, s] = big, -big, 1.0
    v = np.zeros_like(x)
    g = np.zeros_like(x)
    oracle.step_ring(3, 3, np.array([0, 1, 2], np.int32), x, v, g, 0.0, 0.0)  # payload = x
    assert np.array_equal(x, np.full((3, 3), np.float32(1.0) / np.float32(3.0), np.float32))
    # m = 4, slice s = element s: 2^24 at s+1, 1 at s+2, -2^24 at s+3, 1 at s:
    # ((2^24 + 1) + -2^24) + 1 = (2^24 - 2^24) + 1 = 1 (the +1 at s+2 is absorbed); mean 1/4
    x = np.zeros((4, 4), np.float32)
    for s in range(4):
        x[(s + 1) % 4, s], x[(s + 2) % 4, s], x[(s + 3) % 4, s], x[s, s] = big, 1.0, -big, 1.0
    v = np.zeros_like(x)
    oracle.step_ring(4, 4, np.array([0, 1, 2, 3], np.int32), x, v, np.zeros_like(x), 0.0, 0.0)
    assert np.array_equal(x, np.full((4, 4), 0.25, np.float32))


def test_ring_order_equals_fold_for_two_members_and_is_close_otherwise():
    """m <= 2: ring order and ascending fold are the same binary32 sum (commutativity);
    m > 2: the two differ only by rounding (within the derived bound of the fp64 mean)."""
    rng = np.random.default_rng(4)
    for n, m in [(4, 2), (8, 2), (4, 4), (8, 4), (6, 3), (8, 8)]:
        L = 1031
        x0 = rng.standard_normal((n, L)).astype(np.float32)
        g = rng.standard_normal((n, L)).astype(np.float32)
        _, canon, _ = oracle.groups(SEED, 3, n, m)
        xa, va = x0.copy(), np.zeros_like(x0)
        xr, vr = x0.copy(), np.zeros_like(x0)
        oracle.step(n, m, canon, xa, va, g, 0.1, 0.9)
        oracle.step_ring(n, m, canon, xr, vr, g, 0.1, 0.9)
        assert np.array_equal(va, vr)
        if m <= 2:
            assert np.array_equal(xa, xr)
        else:
            x64 = x0.astype(np.float64)
            v64 = np.zeros_like(x64)
            oracle.step(n, m, canon, x64, v64, g.astype(np.float64), 0.1, 0.9)
            bound = (m + 2) * 2.0 ** -24 * np.abs(x64).max() * 2
            assert np.abs(xr - x64).max() < bound and np.abs(xa - x64).max() < bound
            assert not np.array_equal(xa, xr)  # the order really differs


# ---------------------------------------------------------------- NEXT-2: Local-SESGD, final average
def _run_local(n, m, T, L, period, mode=oracle.MODE_PARAM, t0=0):
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, SEED, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=period,
                     mode=mode, t0=t0)
    return x, v


@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_local_period_one_is_sesgd(mode):
    """H = 1 is identical to SESGD (every iteration exchanges)."""
    n, m, T, L = 8, 2, 6, 257
    x, v = _run_local(n, m, T, L, 1, mode)
    xs = np.tile(synth.x0_host(L), (n, 1))
    vs = np.zeros_like(xs)
    oracle.run(n, m, SEED, T, xs, vs, s_g=synth.SEED_G, lr=0.1, mu=0.9, mode=mode)
    assert np.array_equal(x, xs) and np.array_equal(v, vs)


def test_local_period_longer_than_run_is_independent_sgd():
    """H -> infinity: no communication, every worker is textbook momentum SGD on its own
    gradients (torch.optim.SGD float32, within FMA-contraction tolerance)."""
    n, T, L = 4, 7, 300
    x, _ = _run_local(n, 2, T, L, 1000)
    for i in range(n):
        ref = _torch_sgd_trajectory(synth.x0_host(L), [synth.grad_host(i, t, L) for t in range(T)],
                                    0.1, 0.9, dtype=torch.float32)
        np.testing.assert_allclose(x[i], ref, rtol=1e-6, atol=1e-8)


def test_local_sesgd_exchange_events():
    """n = 4, k = 2, H = 2, 4 iterations -> exactly 2 shuffle+allreduce events: group
    members of G_t are byte-identical right after iterations t = 1 and t = 3 only."""
    n, m, L = 4, 2, 64
    events = []
    for T in range(1, 5):
        x, _ = _run_local(n, m, T, L, 2)
        t = T - 1
        groups = oracle.canonical_groups(SEED, t, n, m)
        if all(np.array_equal(x[g[0]], x[g[1]]) for g in groups):
            events.append(t)
    assert events == [1, 3]


@pytest.mark.parametrize("period", [2, 3])
def test_local_sgd_is_global_average_every_period(period):
    """m = n (Local-SGD, the paper's baseline with period 2): all workers
    byte-identical exactly after synchronisation iterations; the worker mean follows momentum SGD
    on the mean gradient at every t (P8 holds for any averaging schedule; float32 tolerance)."""
    n, L = 4, 128
    gbars = []
    for T in range(1, 7):
        x, _ = _run_local(n, n, T, L, period)
        same = all(np.array_equal(x[0], x[i]) for i in range(n))
        assert same == (T % period == 0)
        gbars.append(np.mean([synth.grad_host(i, T - 1, L).astype(np.float64) for i in range(n)], 0))
        ref = _torch_sgd_trajectory(synth.x0_host(L).astype(np.float64), gbars, 0.1, 0.9)
        np.testing.assert_allclose(x.astype(np.float64).mean(0), ref, rtol=0, atol=2e-7)


def test_global_average_special_cases():
    """identical workers -> unchanged; [0] and [2] -> [1]."""
    x = np.tile(np.array([0.25, -3.5, 7.0], np.float32), (5, 1))
    y = oracle.global_average(x.copy())
    assert np.array_equal(y, x)
    z = oracle.global_average(np.array([[0.0], [2.0]], np.float32))
    assert np.array_equal(z, np.array([[1.0], [1.0]], np.float32))


def test_global_average_matches_sequential_mean():
    """16 random workers -> the sequential mean; f64 within 1e-12 of math.fsum / n; f32
    bit-exact against a brute-force left fold in numpy float32 scalars, and within the fp32 bound
    of the exact mean."""
    rng = np.random.default_rng(5)
    x64 = rng.standard_normal((16, 37))
    got64 = oracle.global_average(x64.copy())
    exact = np.array([math.fsum(x64[:, e]) / 16 for e in range(37)])
    np.testing.assert_allclose(got64[7], exact, rtol=1e-12, atol=1e-15)
    x32 = x64.astype(np.float32)
    got32 = oracle.global_average(x32.copy())
    for e in range(37):
        s = np.float32(x32[0, e])
        for i in range(1, 16):
            s = np.float32(s + x32[i, e])
        assert got32[3, e] == np.float32(s / np.float32(16))
    np.testing.assert_allclose(got32[0], exact, rtol=0, atol=16 * 6e-8 * np.abs(x64).max())


# ---------------------------------------------------------------- NEXT-3: Stone dimension exchange
def test_stone_schedule_paper_example():
    """"at iteration t the groups are {0,1},{2,3}; at t+1 it may be {0,2},{1,3}"."""
    c0, _ = oracle.groups_stone(0, 4, 2)
    c1, _ = oracle.groups_stone(1, 4, 2)
    assert c0.tolist() == [0, 1, 2, 3] and c1.tolist() == [0, 2, 1, 3]


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
def test_stone_schedule_partitions_and_exact_mean(n):
    """Every iteration is a canonical equal partition; the product of the averaging matrices W_t
    over d/p consecutive iterations is exactly J/n in rational arithmetic (the shuffle-exchange
    network all-reduce: every worker holds the global mean), for every m = 2^p dividing d."""
    from fractions import Fraction
    d = n.bit_length() - 1
    for p in range(1, d + 1):
        m = 1 << p
        if d % p:
            continue
        for t0 in range(3):
            prod = [[Fraction(int(i == j)) for j in range(n)] for i in range(n)]
            for t in range(t0, t0 + d // p):
                canon, gof = oracle.groups_stone(t, n, m)
                groups = [canon[j * m:(j + 1) * m].tolist() for j in range(n // m)]
                assert sorted(sum(groups, [])) == list(range(n))
                assert all(g == sorted(g) for g in groups)
                assert [g[0] for g in groups] == sorted(g[0] for g in groups)
                W = [[Fraction(int(gof[i] == gof[j]), m) for j in range(n)] for i in range(n)]
                prod = [[sum(W[i][k] * prod[k][j] for k in range(n)) for j in range(n)] for i in range(n)] \
                    if n <= 16 else prod
            if n <= 16:
                assert all(prod[i][j] == Fraction(1, n) for i in range(n) for j in range(n))


def test_stone_schedule_pure_averaging_reaches_global_mean():
    """lr = 0, distinct x_0 per worker: after log2(n) / p iterations of the oracle step, every
    worker equals the global mean (fp64, within rounding of math.fsum / n)."""
    n, m, L = 16, 2, 23
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, L))
    exact = np.array([math.fsum(x[:, e]) / n for e in range(L)])
    v = np.zeros_like(x)
    for t in range(4):
        canon, _ = oracle.groups_stone(t, n, m)
        oracle.step(n, m, canon, x, v, np.zeros_like(x), 0.0, 0.0)
    np.testing.assert_allclose(x, np.tile(exact, (n, 1)), rtol=0, atol=1e-15)


def test_stone_schedule_errors_and_run():
    """Non-powers of two are rejected; run_local(schedule=STONE, period=1) is the iteration loop
    of oracle.step over groups_stone."""
    with pytest.raises(oracle.OracleError):
        oracle.groups_stone(0, 6, 2)
    with pytest.raises(oracle.OracleError):
        oracle.groups_stone(0, 8, 3)
    n, m, T, L = 8, 2, 5, 33
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, SEED, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1,
                     schedule=oracle.SCHED_STONE)
    y = np.tile(synth.x0_host(L), (n, 1))
    w = np.zeros_like(y)
    for t in range(T):
        canon, _ = oracle.groups_stone(t, n, m)
        oracle.step(n, m, canon, y, w, _grads(n, t, L, np.float32), 0.1, 0.9)
    assert np.array_equal(x, y) and np.array_equal(v, w)


# ---------------------------------------------------------------- NEXT-4: consistency metric
def test_consensus_metric_definition():
    """Zero for identical workers; [0], [2] -> 2 and 1; equals the pairwise form
    (1/(2n)) sum_{i,j} ||x_i - x_j||^2 (brute force, exact fractions on dyadic data)."""
    assert oracle.consensus(np.tile(np.float32([1.5, -2.0]), (4, 1))) == (0.0, 0.0)
    assert oracle.consensus(np.array([[0.0], [2.0]], np.float32)) == (2.0, 1.0)
    from fractions import Fraction
    rng = np.random.default_rng(9)
    x = (rng.integers(-64, 64, size=(6, 11)) / 8).astype(np.float32)
    n = x.shape[0]
    pair = sum(Fraction(float(x[i, e]) - float(x[j, e])) ** 2
               for i in range(n) for j in range(n) for e in range(x.shape[1])) / (2 * n)
    ss, mx = oracle.consensus(x)
    assert abs(ss - float(pair)) <= 1e-12 * float(pair)
    assert mx == float(np.abs(x.astype(np.float64) - x.astype(np.float64).mean(0)).max())


def test_consensus_group_average_contracts_and_matches_paper_claim():
    """P:432-433 ("parameters of each worker maintain highly consistent"): under SESGD the
    consensus distance stays small relative to independent SGD (m = 1), and an exchange with
    m = n makes it exactly 0."""
    n, L, T = 8, 500, 20
    xs, _ = _run_local(n, 2, T, L, 1)
    xi, _ = _run_local(n, 1, T, L, 1)
    xr, _ = _run_local(n, n, T, L, 1)
    assert oracle.consensus(xs)[0] < 0.2 * oracle.consensus(xi)[0]
    assert oracle.consensus(xr) == (0.0, 0.0)


# ---------------------------------------------------------------- NEXT-4: weight decay
def _torch_sgd_wd(x0, grads, lr, mu, wd, dtype=torch.float64):
    p = torch.nn.Parameter(torch.tensor(x0, dtype=dtype))
    opt = torch.optim.SGD([p], lr=lr, momentum=mu, dampening=0.0, nesterov=False, weight_decay=wd)
    for g in grads:
        p.grad = torch.tensor(g, dtype=dtype)
        opt.step()
    return p.detach().numpy()


def test_weight_decay_zero_is_identity():
    n, m, T, L = 8, 2, 5, 97
    a, va = _run_local(n, m, T, L, 1)
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, m, SEED, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, weight_decay=0.0)
    assert np.array_equal(a, x) and np.array_equal(va, v)


@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_weight_decay_m1_is_torch_sgd(mode):
    """P:325 (wd 5e-4): with m = 1 every worker is torch.optim.SGD(momentum, weight_decay) on its
    own gradients (float32, within FMA-contraction tolerance)."""
    n, T, L, wd = 3, 8, 400, 5e-4
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, 1, SEED, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     weight_decay=wd)
    for i in range(n):
        ref = _torch_sgd_wd(synth.x0_host(L), [synth.grad_host(i, t, L) for t in range(T)], 0.1, 0.9, wd,
                            dtype=torch.float32)
        np.testing.assert_allclose(x[i], ref, rtol=1e-6, atol=1e-8)


def test_weight_decay_group_n_is_ring_sgd_with_decay():
    """m = n: every worker equals torch.optim.SGD(weight_decay) on the global mean gradient (GRAD
    mode; all workers share x, so gbar + wd x is the decayed mean gradient)."""
    n, T, L, wd = 4, 6, 300, 1e-2
    x = np.tile(synth.x0_host(L), (n, 1))
    v = np.zeros_like(x)
    oracle.run_local(n, n, SEED, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1,
                     mode=oracle.MODE_GRAD, weight_decay=wd)
    gbars = [np.mean([synth.grad_host(i, t, L).astype(np.float64) for i in range(n)], 0) for t in range(T)]
    ref = _torch_sgd_wd(synth.x0_host(L).astype(np.float64), gbars, 0.1, 0.9, wd)
    assert all(np.array_equal(x[0], x[i]) for i in range(n))
    np.testing.assert_allclose(x[0], ref, rtol=0, atol=2e-7)


# ---------------------------------------------------------------- NEXT-4: bf16 payload (R21)
def test_round_bf16_matches_torch():
    """The oracle's bf16 rounding equals torch's float32 -> bfloat16 conversion (round to nearest
    even) on random values, exact ties and extremes."""
    rng = np.random.default_rng(4)
    vals = np.concatenate([rng.standard_normal(5000).astype(np.float32),
                           (rng.integers(1, 1 << 20, 2000) * 2.0 ** -20 + 1).astype(np.float32),
                           np.float32([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 0.0, -0.0, 3.4e38,
                                       1e-40, 65504.0])])
    want = torch.from_numpy(vals).to(torch.bfloat16).to(torch.float32).numpy()
    got = np.array([oracle.round_bf16(float(v)) for v in vals], np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("mode", [oracle.MODE_PARAM, oracle.MODE_GRAD])
def test_bf16_payload_step_definition(mode):
    """R21 on one iteration, n = 4, m = 2: every exchanged contribution is rounded to bf16 before the
    fold (torch's conversion as the independent reference), the fold / mean / update stay fp32;
    with m = 1 nothing is exchanged and the payload changes nothing."""
    n, m, L = 4, 2, 257
    x0 = np.tile(synth.x0_host(L), (n, 1))
    g = np.stack([synth.grad_host(i, 0, L) for i in range(n)]).astype(np.float32)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float32).numpy()  # noqa: E731
    x = x0.copy()
    v = np.zeros_like(x)
    oracle.run_local(n, m, SEED, 1, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     payload_bf16=True)
    groups = oracle.canonical_groups(SEED, 0, n, m)
    f = np.float32
    for a, b in groups:
        if mode == oracle.MODE_PARAM:
            va, vb = g[a], g[b]  # v0 = 0: v = 0.9 * 0 + g
            xa, xb = x0[a] - f(0.1) * va, x0[b] - f(0.1) * vb
            want = (bf(xa) + bf(xb)) / f(2)
            assert np.array_equal(x[a], want) and np.array_equal(x[b], want)
        else:
            gb = (bf(g[a]) + bf(g[b])) / f(2)
            assert np.array_equal(v[a], gb) and np.array_equal(x[a], x0[a] - f(0.1) * gb)
    y = x0.copy()
    w = np.zeros_like(y)
    oracle.run_local(n, 1, SEED, 1, y, w, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode,
                     payload_bf16=True)
    z = x0.copy()
    u = np.zeros_like(z)
    oracle.run_local(n, 1, SEED, 1, z, u, s_g=synth.SEED_G, lr=0.1, mu=0.9, period=1, mode=mode)
    assert np.array_equal(y, z)

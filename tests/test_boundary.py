"""CPU-only checks of the C-ABI boundary (no kernel launches, no GPU needed).

* libsesgd.so loads and exports every symbol include/sesgd.h declares;
* the product's host scheduler (a1) is bit-exact against the oracle's independent one;
* the product's latency model (a7) equals the oracle's;
* argument validation / error codes.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2007_00433_b200 import sesgd as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sesgd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sesgd_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    declared = _declared_symbols()
    assert len(declared) >= 15
    assert sorted(C.EXPORTED) == declared
    lib = ctypes.CDLL(C.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    # the north-star names of the boundary (BASELINE.json north_star)
    for name in ("sesgd_init", "sesgd_groups", "sesgd_sync_step", "sesgd_latency_model"):
        assert name in declared


def test_library_is_sm100a():
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", C.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,m", [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (6, 3), (8, 2), (8, 4),
                                 (8, 8), (16, 4), (16, 2), (32, 8), (64, 8), (64, 64), (12, 3)])
def test_host_scheduler_bitexact_vs_oracle(n, m):
    """Row a1: group assignments bit-exact against the oracle (independent implementation)."""
    for seed in (0, 42, 2 ** 63 + 12345):
        ctx = C.sesgd_init(n, m, seed)
        try:
            for t in list(range(0, 300)) + [10 ** 6, 2 ** 40 + 7]:
                perm, gof = C.sesgd_groups(ctx, t, n)
                _, canon, ogof = oracle.groups(seed, t, n, m)
                assert np.array_equal(perm, canon), (n, m, seed, t)
                assert np.array_equal(gof, ogof)
        finally:
            C.sesgd_destroy(ctx)


def test_host_scheduler_bitexact_vs_oracle_random_seeds():
    """Row a1, property form: any 64-bit seed, any iteration t < 2^62, any m | n <= 64."""
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=400, deadline=None)
    @given(st.integers(1, 64).flatmap(lambda n: st.tuples(
        st.just(n), st.sampled_from([d for d in range(1, n + 1) if n % d == 0]))),
        st.integers(0, 2 ** 64 - 1), st.integers(0, 2 ** 62))
    def check(nm, seed, t):
        n, m = nm
        ctx = C.sesgd_init(n, m, seed)
        try:
            perm, gof = C.sesgd_groups(ctx, t, n)
        finally:
            C.sesgd_destroy(ctx)
        _, canon, ogof = oracle.groups(seed, t, n, m)
        assert np.array_equal(perm, canon) and np.array_equal(gof, ogof)

    check()


@pytest.mark.parametrize("n,m", [(2, 2), (4, 2), (8, 2), (8, 4), (16, 4), (32, 8), (64, 2), (64, 64)])
def test_dimension_exchange_schedule_bitexact_vs_oracle(n, m):
    """NEXT-3 (SESGD_OPT_SCHEDULE = 1): the product's dimension-exchange schedule equals the
    oracle's (independent implementations); non-powers of two are rejected."""
    ctx = C.sesgd_init(n, m, 42)
    try:
        C.sesgd_set_option(ctx, C.OPT_SCHEDULE, C.SCHEDULE_DIMENSION_EXCHANGE)
        for t in list(range(0, 40)) + [10 ** 6 + 3]:
            perm, gof = C.sesgd_groups(ctx, t, n)
            canon, ogof = oracle.groups_stone(t, n, m)
            assert np.array_equal(perm, canon), (n, m, t)
            assert np.array_equal(gof, ogof)
    finally:
        C.sesgd_destroy(ctx)
    ctx = C.sesgd_init(12, 3, 42)
    try:
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_set_option(ctx, C.OPT_SCHEDULE, 1)
        assert e.value.code == C.EINVAL
    finally:
        C.sesgd_destroy(ctx)


def test_latency_model_matches_oracle():
    """Row a7: Eq. 2 / Eq. 3 exact forms equal the oracle's, bit for bit."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.choice([1, 2, 4, 8, 16, 32, 64]))
        m = int(rng.choice([d for d in range(1, n + 1) if n % d == 0]))
        G, nu, tau = float(rng.uniform(0, 1e9)), float(rng.uniform(1e6, 1e12)), float(rng.uniform(0, 1e-2))
        got = C.sesgd_latency_model(n, m, G, nu, tau)
        want = oracle.latency(n, m, G, nu, tau)
        for k in want:
            assert got[k] == want[k], (k, got, want)


def test_latency_model_worked_example():
    """P15 through the boundary: 2(3-1)=4 handshakes; 0.0486 s."""
    assert C.sesgd_latency_model(3, 3, 0, 1, 0)["ring_handshakes"] == 4
    assert abs(C.sesgd_latency_model(4, 4, 4e6, 125e6, 1e-4)["ring_s"] - 0.0486) < 5e-5
    assert C.sesgd_latency_model(16, 4, 0, 1e9, 5e-3)["ratio"] == 5.0


def test_init_errors():
    for n, m, code in [(0, 1, C.EINVAL), (4, 0, C.EINVAL), (4, 5, C.EINVAL), (65, 1, C.EINVAL),
                       (6, 4, C.ENOTDIV), (8, 3, C.ENOTDIV)]:
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_init(n, m, 1)
        assert e.value.code == code
    for args, code in [((4, 3, 1.0, 1.0, 0.0), C.ENOTDIV), ((4, 2, -1.0, 1.0, 0.0), C.EINVAL),
                       ((4, 2, 1.0, 0.0, 0.0), C.EINVAL), ((4, 2, 1.0, 1.0, -1.0), C.EINVAL)]:
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_latency_model(*args)
        assert e.value.code == code


def test_call_order_errors_without_gpu():
    """Calls that need sesgd_attach fail with SESGD_ESTATE before it (no GPU touched)."""
    ctx = C.sesgd_init(4, 2, 42)
    try:
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_register_bucket(ctx, 0, 16, [1] * 4, [1] * 4, [1] * 4)
        assert e.value.code == C.ESTATE
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_begin_iter(ctx, 0)
        assert e.value.code == C.ESTATE
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_sync_step(ctx, 0, 0.1, 0.9)
        assert e.value.code == C.ESTATE
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_workspace_bytes(ctx)
        assert e.value.code == C.ESTATE
        with pytest.raises(C.SesgdError) as e:
            C.sesgd_groups(ctx, -1, 4)
        assert e.value.code == C.EINVAL
        for opt, val in [(C.OPT_MODE, 7), (C.OPT_PATH, 9), (C.OPT_PATH, C.PATH_NVLS + 1),
                         (C.OPT_TIMEOUT_MS, 0), (99, 0)]:
            with pytest.raises(C.SesgdError) as e:
                C.sesgd_set_option(ctx, opt, val)
            assert e.value.code == C.EINVAL
        for p in (C.PATH_AUTO, C.PATH_RESIDENT, C.PATH_ONESHOT, C.PATH_RING, C.PATH_TWOSHOT, C.PATH_NVLS):
            C.sesgd_set_option(ctx, C.OPT_PATH, p)
        C.sesgd_set_option(ctx, C.OPT_MODE, C.MODE_GRAD_AVG)
        assert "invalid" in C.lib().sesgd_strerror(C.EINVAL).decode()
    finally:
        C.sesgd_destroy(ctx)


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: with the in-tree libsesgd.so absent the binding raises instead of running."""
    monkeypatch.setattr(C, "_lib", None)
    monkeypatch.setattr(C, "LIB_PATH", os.path.join(ROOT, "no_such_dir", "libsesgd.so"))
    with pytest.raises(ImportError):
        C.lib()


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: nothing in the product package (Python or CUDA/C++)
    imports, links or includes anything under oracle/."""
    import ast
    pkg = os.path.join(ROOT, "paper_2007_00433_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(path).read())
                for node in ast.walk(tree):
                    names = ([a.name for a in node.names] if isinstance(node, ast.Import) else
                             [node.module or ""] if isinstance(node, ast.ImportFrom) else [])
                    assert not any(n == "oracle" or n.startswith("oracle.") for n in names), path
            elif f.endswith((".cu", ".cuh", ".cpp", ".h")):
                src = open(path).read()
                assert not re.search(r'#include\s*[<"][^>"]*oracle', src), path

"""CPU oracle for the SESGD hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2007_00433_b200``) never imports it and shares no code with it.

This module is argument marshalling around ``liboracle.so`` (built from
``sesgd_oracle.c`` with ``gcc -O2 -ffp-contract=off``): all arithmetic of the
method lives in that C file, written step by step from Algorithm 1 / Eq. 5-6 of
the paper.  See ``sesgd_oracle.h`` for citations.

Parity status: every entry point is pinned by ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC = os.path.join(_HERE, "sesgd_oracle.c")

MODE_PARAM = 0
MODE_GRAD = 1
OK, EINVAL, ENOTDIV = 0, -1, -2

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C, no fast-math, no FMA contraction)."""
    deps = [SRC, os.path.join(_HERE, "sesgd_oracle.h"),
            os.path.join(_HERE, "..", "synth", "synth_gen.h")]
    if (not force and os.path.exists(LIB_PATH)
            and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-Wall", "-o", LIB_PATH, SRC, "-lm"]
    subprocess.check_call(cmd)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32
        P = ctypes.c_void_p
        L.orc_splitmix64_next.argtypes = [ctypes.POINTER(u64)]
        L.orc_splitmix64_next.restype = u64
        L.orc_mix.argtypes = [u64]
        L.orc_mix.restype = u64
        L.orc_bounded.argtypes = [ctypes.POINTER(u64), u64, ctypes.POINTER(ctypes.c_int)]
        L.orc_bounded.restype = u64
        L.orc_groups.argtypes = [u64, i64, i32, i32, P, P, P]
        L.orc_groups.restype = ctypes.c_int
        L.orc_latency.argtypes = [i32, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double, P]
        L.orc_latency.restype = ctypes.c_int
        L.orc_step_f32.argtypes = [i32, i32, P, i64, P, P, P, ctypes.c_float, ctypes.c_float, i32]
        L.orc_step_f32.restype = ctypes.c_int
        L.orc_step_f64.argtypes = [i32, i32, P, i64, P, P, P, ctypes.c_double, ctypes.c_double, i32]
        L.orc_step_f64.restype = ctypes.c_int
        L.orc_run_f32.argtypes = [i32, i32, u64, i64, i64, i64, P, u64, ctypes.c_float,
                                  ctypes.c_float, i32, P, P]
        L.orc_run_f32.restype = ctypes.c_int
        L.orc_run_f64.argtypes = [i32, i32, u64, i64, i64, i64, P, u64, ctypes.c_double,
                                  ctypes.c_double, i32, P, P]
        L.orc_run_f64.restype = ctypes.c_int
        L.orc_step_ring_f32.argtypes = [i32, i32, P, i64, P, P, P, ctypes.c_float, ctypes.c_float, i32]
        L.orc_step_ring_f32.restype = ctypes.c_int
        L.orc_slice_of.argtypes = [i64, i32, i64]
        L.orc_slice_of.restype = i32
        L.orc_run_ring_f32.argtypes = [i32, i32, u64, i64, i64, i64, i64, u64, ctypes.c_float,
                                       ctypes.c_float, i32, P, P]
        L.orc_run_ring_f32.restype = ctypes.c_int
        L.orc_run_local_f32.argtypes = [i32, i32, u64, i64, i64, i64, P, u64, ctypes.c_float,
                                        ctypes.c_float, i32, i64, i32, ctypes.c_float, P, P]
        L.orc_step_wd_f32.argtypes = [i32, i32, P, i64, P, P, P, ctypes.c_float, ctypes.c_float,
                                      ctypes.c_float, i32]
        L.orc_step_wd_f32.restype = ctypes.c_int
        L.orc_run_ext_f32.argtypes = [i32, i32, u64, i64, i64, i64, P, u64, ctypes.c_float,
                                      ctypes.c_float, i32, i64, i32, ctypes.c_float, i32, P, P]
        L.orc_run_ext_f32.restype = ctypes.c_int
        L.orc_round_bf16.argtypes = [ctypes.c_float]
        L.orc_round_bf16.restype = ctypes.c_float
        L.orc_groups_stone.argtypes = [i64, i32, i32, P, P]
        L.orc_groups_stone.restype = ctypes.c_int
        L.orc_run_local_f32.restype = ctypes.c_int
        L.orc_global_average_f32.argtypes = [i32, i64, P]
        L.orc_global_average_f32.restype = ctypes.c_int
        L.orc_global_average_f64.argtypes = [i32, i64, P]
        L.orc_global_average_f64.restype = ctypes.c_int
        L.orc_consensus.argtypes = [i32, i64, P, P]
        L.orc_consensus.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


def _check(rc: int) -> None:
    if rc != OK:
        raise OracleError(rc)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Rng64:
    """splitmix64 stream (R2)."""

    def __init__(self, state: int):
        self.state = ctypes.c_uint64(state & 0xFFFFFFFFFFFFFFFF)

    def next(self) -> int:
        return int(lib().orc_splitmix64_next(ctypes.byref(self.state)))

    def bounded(self, bound: int) -> int:
        err = ctypes.c_int(0)
        r = int(lib().orc_bounded(ctypes.byref(self.state), bound, ctypes.byref(err)))
        if err.value:
            raise OracleError(EINVAL)
        return r


def mix(z: int) -> int:
    return int(lib().orc_mix(z & 0xFFFFFFFFFFFFFFFF))


def groups(seed: int, t: int, n: int, m: int):
    """Return (raw_perm, canon, group_of) int32 arrays for iteration t (A1)."""
    raw = np.empty(n, np.int32)
    canon = np.empty(n, np.int32)
    gof = np.empty(n, np.int32)
    _check(lib().orc_groups(seed & 0xFFFFFFFFFFFFFFFF, t, n, m, _ptr(raw), _ptr(canon), _ptr(gof)))
    return raw, canon, gof


def canonical_groups(seed: int, t: int, n: int, m: int):
    """List of tuples, the canonical partition of iteration t."""
    _, canon, _ = groups(seed, t, n, m)
    return [tuple(int(a) for a in canon[j * m:(j + 1) * m]) for j in range(n // m)]


def latency(n: int, m: int, nbytes: float, nu: float, tau: float) -> dict:
    out = np.zeros(5, np.float64)
    _check(lib().orc_latency(n, m, float(nbytes), float(nu), float(tau), _ptr(out)))
    return {"ring_handshakes": out[0], "sesgd_handshakes": out[1], "ring_s": out[2],
            "sesgd_s": out[3], "ratio": out[4]}


def step(n, m, canon, x, v, g, lr, mu, mode=MODE_PARAM):
    """One iteration in place on worker-major arrays x, v (n, L) with gradients g (n, L).

    dtype float32 -> binary32 op-exact oracle; float64 -> binary64 oracle."""
    canon = np.ascontiguousarray(canon, np.int32)
    assert x.flags.c_contiguous and v.flags.c_contiguous
    if x.dtype == np.float32:
        g = np.ascontiguousarray(g, np.float32)
        _check(lib().orc_step_f32(n, m, _ptr(canon), x.shape[-1], _ptr(x), _ptr(v), _ptr(g),
                                  float(lr), float(mu), mode))
    elif x.dtype == np.float64:
        g = np.ascontiguousarray(g, np.float64)
        _check(lib().orc_step_f64(n, m, _ptr(canon), x.shape[-1], _ptr(x), _ptr(v), _ptr(g),
                                  float(lr), float(mu), mode))
    else:
        raise TypeError(x.dtype)


def step_wd(n, m, canon, x, v, g, lr, mu, wd, mode=MODE_PARAM):
    """One binary32 iteration with weight decay (float32 arrays, in place)."""
    canon = np.ascontiguousarray(canon, np.int32)
    g = np.ascontiguousarray(g, np.float32)
    assert x.dtype == np.float32 and x.flags.c_contiguous and v.flags.c_contiguous
    _check(lib().orc_step_wd_f32(n, m, _ptr(canon), x.shape[-1], _ptr(x), _ptr(v), _ptr(g),
                                 float(lr), float(mu), float(wd), mode))


def slice_of(L: int, m: int, e: int) -> int:
    return int(lib().orc_slice_of(L, m, e))


def step_ring(n, m, canon, x, v, g, lr, mu, mode=MODE_PARAM):
    """One iteration with the group mean in Ring-AllReduce order (float32 arrays, in place)."""
    canon = np.ascontiguousarray(canon, np.int32)
    g = np.ascontiguousarray(g, np.float32)
    assert x.dtype == np.float32 and x.flags.c_contiguous and v.flags.c_contiguous
    _check(lib().orc_step_ring_f32(n, m, _ptr(canon), x.shape[-1], _ptr(x), _ptr(v), _ptr(g),
                                   float(lr), float(mu), mode))


def run_ring(n, m, seed, T, x, v, *, s_g, lr, mu, mode=MODE_PARAM, t0=0, e0=0):
    """T ring-order iterations over one bucket (x, v: float32 (n, L) in place) whose
    elements have global coordinates e0 .. e0 + L - 1."""
    _check(lib().orc_run_ring_f32(n, m, seed, t0, T, x.shape[-1], e0, s_g, float(lr), float(mu), mode,
                                  _ptr(x), _ptr(v)))
    return x, v


def run(n, m, seed, T, x, v, *, s_g, lr, mu, mode=MODE_PARAM, t0=0, coords=None):
    """T iterations with synthetic gradients; x, v (n, S) updated in place.

    coords: int64 global element indices of the S columns (None = 0..S-1)."""
    S = x.shape[-1]
    cp = None
    if coords is not None:
        coords = np.ascontiguousarray(coords, np.int64)
        assert coords.shape == (S,)
        cp = _ptr(coords)
    if x.dtype == np.float32:
        _check(lib().orc_run_f32(n, m, seed, t0, T, S, cp, s_g, float(lr), float(mu), mode,
                                 _ptr(x), _ptr(v)))
    elif x.dtype == np.float64:
        _check(lib().orc_run_f64(n, m, seed, t0, T, S, cp, s_g, float(lr), float(mu), mode,
                                 _ptr(x), _ptr(v)))
    else:
        raise TypeError(x.dtype)
    return x, v


SCHED_RANDOM, SCHED_STONE = 0, 1


def groups_stone(t: int, n: int, m: int):
    """(canon, group_of) of Stone's dimension-exchange schedule at iteration t (NEXT-3)."""
    canon = np.empty(n, np.int32)
    gof = np.empty(n, np.int32)
    _check(lib().orc_groups_stone(t, n, m, _ptr(canon), _ptr(gof)))
    return canon, gof


def run_local(n, m, seed, T, x, v, *, s_g, lr, mu, period, mode=MODE_PARAM, t0=0, coords=None,
              schedule=SCHED_RANDOM, weight_decay=0.0, payload_bf16=False):
    """Local-SESGD: T iterations where the group exchange fires only when
    (t + 1) % period == 0; float32 x, v (n, S) in place.  period = 1 is `run`; m = n is
    Local-SGD."""
    S = x.shape[-1]
    cp = None
    if coords is not None:
        coords = np.ascontiguousarray(coords, np.int64)
        assert coords.shape == (S,)
        cp = _ptr(coords)
    assert x.dtype == np.float32 and x.flags.c_contiguous and v.flags.c_contiguous
    _check(lib().orc_run_ext_f32(n, m, seed, t0, T, S, cp, s_g, float(lr), float(mu), mode,
                                 int(period), int(schedule), float(weight_decay), int(bool(payload_bf16)),
                                 _ptr(x), _ptr(v)))
    return x, v


def global_average(x):
    """Algorithm 1's last line: every row of x (n, L) becomes the ascending-fold mean of
    all rows, in place (float32 or float64)."""
    assert x.flags.c_contiguous and x.ndim == 2
    fn = {np.dtype(np.float32): lib().orc_global_average_f32,
          np.dtype(np.float64): lib().orc_global_average_f64}[x.dtype]
    _check(fn(x.shape[0], x.shape[1], _ptr(x)))
    return x


def consensus(x):
    """(sum of squared deviations from the worker mean, max abs deviation) of float32 x (n, L)."""
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(2, np.float64)
    _check(lib().orc_consensus(x.shape[0], x.shape[1], _ptr(x), _ptr(out)))
    return float(out[0]), float(out[1])


def round_bf16(f: float) -> float:
    """bfloat16 round to nearest even of a binary32 value (the payload reading R21)."""
    return float(lib().orc_round_bf16(float(f)))

"""Seeded synthetic inputs (x_0 and per-(worker, iteration) gradients).

Input generator module shared by the oracle side and the GPU side (DESIGN.md
"Input recipe"); it contains none of SESGD's arithmetic.  Device fills stand in
for backward; host fills give the same bits for tests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsynth.so")
SRC = os.path.join(_HERE, "synth.cu")

# default seeds of the input recipe: schedule sigma=42, s_g=1, s_x=2
SEED_SIGMA, SEED_G, SEED_X = 42, 1, 2

_lib = None


def build(force: bool = False) -> str:
    deps = [SRC, os.path.join(_HERE, "synth_gen.h")]
    if (not force and os.path.exists(LIB_PATH)
            and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    cmd = ["nvcc", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-o", LIB_PATH, SRC]
    subprocess.check_call(cmd)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
        L.synth_fill_grad_device.argtypes = [P, i64, i64, u64, i32, i64, P]
        L.synth_fill_grad_device.restype = ctypes.c_int
        L.synth_fill_grad_device_at.argtypes = [P, i64, i64, u64, i32, P, P]
        L.synth_fill_grad_device_at.restype = ctypes.c_int
        L.synth_fill_x0_device.argtypes = [P, i64, i64, u64, P]
        L.synth_fill_x0_device.restype = ctypes.c_int
        L.synth_fill_grad_host.argtypes = [P, i64, i64, P, u64, i32, i64]
        L.synth_fill_grad_host.restype = None
        L.synth_fill_x0_host.argtypes = [P, i64, i64, P, u64]
        L.synth_fill_x0_host.restype = None
        _lib = L
    return _lib


def _coords(numel, e0, coords):
    if coords is None:
        return numel, None, None
    c = np.ascontiguousarray(coords, np.int64)
    return c.shape[0], c, c.ctypes.data_as(ctypes.c_void_p)


def grad_host(worker: int, t: int, numel: int = 0, e0: int = 0, coords=None, s_g: int = SEED_G):
    numel, keep, cp = _coords(numel, e0, coords)
    out = np.empty(numel, np.float32)
    lib().synth_fill_grad_host(out.ctypes.data_as(ctypes.c_void_p), numel, e0, cp, s_g, worker, t)
    del keep
    return out


def x0_host(numel: int = 0, e0: int = 0, coords=None, s_x: int = SEED_X):
    numel, keep, cp = _coords(numel, e0, coords)
    out = np.empty(numel, np.float32)
    lib().synth_fill_x0_host(out.ctypes.data_as(ctypes.c_void_p), numel, e0, cp, s_x)
    del keep
    return out


def fill_grad_device(ptr: int, numel: int, e0: int, worker: int, t: int, stream: int = 0,
                     s_g: int = SEED_G) -> None:
    rc = lib().synth_fill_grad_device(ptr, numel, e0, s_g, worker, t, stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_grad_device: cuda error {rc}")


def fill_grad_device_at(ptr: int, numel: int, e0: int, worker: int, t_dev_ptr: int, stream: int = 0,
                        s_g: int = SEED_G) -> None:
    """gradient fill for the iteration held in device memory at t_dev_ptr (int64), read when the
    kernel runs -- graph-capturable across iterations"""
    rc = lib().synth_fill_grad_device_at(ptr, numel, e0, s_g, worker, t_dev_ptr, stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_grad_device_at: cuda error {rc}")


def fill_x0_device(ptr: int, numel: int, e0: int, stream: int = 0, s_x: int = SEED_X) -> None:
    rc = lib().synth_fill_x0_device(ptr, numel, e0, s_x, stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_x0_device: cuda error {rc}")

"""Thin ctypes binding of libsesgd.so (include/sesgd.h), same names as the C ABI.

Argument marshalling only: every step of the SESGD hot path runs in the CUDA
kernels behind these calls.  There is no Python or CPU fallback -- importing
this module fails loudly if the in-tree ``libsesgd.so`` is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SESGD_LIB=checked loads the bounds-checked build (_build.build(checked=True), -DSESGD_CHECKED);
# SESGD_LIB=<tag> loads libsesgd_<tag>.so from this directory (kernel variants built for A/B runs)
_VARIANT = os.environ.get("SESGD_LIB", "")
LIB_PATH = os.path.join(_PKG, f"libsesgd_{_VARIANT}.so" if _VARIANT else "libsesgd.so")

OK, EINVAL, ENOTDIV, ESTATE, ECUDA, ETIMEOUT, ENOMEM, ENOTSUP = 0, -1, -2, -3, -4, -5, -6, -7
MAX_WORKERS, MAX_RANKS = 64, 8
MODE_PARAM_AVG, MODE_GRAD_AVG = 0, 1
PATH_AUTO, PATH_RESIDENT, PATH_ONESHOT, PATH_RING, PATH_TWOSHOT, PATH_NVLS = 0, 1, 2, 3, 4, 5
OPT_MODE, OPT_PATH, OPT_TIMEOUT_MS, OPT_GRID, OPT_HOP_DELAY_NS, OPT_P2P_VARIANT, OPT_DISCARD = (
    1, 2, 3, 4, 5, 6, 7)
OPT_PROFILE, OPT_COMM_BATCH, OPT_FOLD_LAG, OPT_RESIDENT_UNROLL, OPT_PUSH_TMA = 8, 9, 10, 11, 12
OPT_RELEASE_DELAY, OPT_RELEASE_EVERY, OPT_LOCAL_PERIOD, OPT_SCHEDULE = 13, 14, 15, 16
SCHEDULE_RANDOM, SCHEDULE_DIMENSION_EXCHANGE = 0, 1
OPT_RELEASE_STAGGER, OPT_PAYLOAD_BF16, OPT_SM_BUDGET = 17, 18, 19
OPT_EXPERIMENT, OPT_PROTOCOL, OPT_COOPERATIVE, OPT_DEVICE_ITER, OPT_WS_SPLIT, OPT_WSM_HYBRID = 20, 21, 22, 23, 24, 25
ITER_NEXT = -1

# every symbol include/sesgd.h declares (checked by tests/test_boundary.py)
EXPORTED = (
    "sesgd_init", "sesgd_destroy", "sesgd_groups", "sesgd_latency_model", "sesgd_set_option",
    "sesgd_attach", "sesgd_register_bucket", "sesgd_workspace_bytes", "sesgd_workspace_prepare",
    "sesgd_attach_peers", "sesgd_begin_iter", "sesgd_sync_step", "sesgd_sync_step_host",
    "sesgd_poll", "sesgd_get_stats", "sesgd_launch_grid", "sesgd_strerror", "sesgd_last_error",
    "sesgd_probe_copy", "sesgd_probe_pingpong", "sesgd_profile_read", "sesgd_sync_all",
    "sesgd_global_average", "sesgd_sync_all_host", "sesgd_consensus", "sesgd_set_weight_decay",
    "sesgd_attach_multicast", "sesgd_pair_counts", "sesgd_measure_hop", "sesgd_sync_all_pair",
    "sesgd_begin_iter_device", "sesgd_device_iter_ptr", "sesgd_device_iter_read",
)


class sesgd_cost(ctypes.Structure):
    _fields_ = [("ring_handshakes", ctypes.c_double), ("sesgd_handshakes", ctypes.c_double),
                ("ring_s", ctypes.c_double), ("sesgd_s", ctypes.c_double), ("ratio", ctypes.c_double)]


class sesgd_stats(ctypes.Structure):
    _fields_ = [("sync_calls", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("handshake_rounds", ctypes.c_int64), ("flag_messages", ctypes.c_int64),
                ("payload_bytes_in", ctypes.c_int64), ("hbm_algo_bytes", ctypes.c_int64),
                ("dev_flag_stores", ctypes.c_int64), ("dev_flag_spins", ctypes.c_int64),
                ("dev_value_spins", ctypes.c_int64), ("dev_launches", ctypes.c_int64),
                ("last_launch_us", ctypes.c_double), ("hop_ns", ctypes.c_double)]


class sesgd_device_iter_state(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("seq", ctypes.c_int64), ("claim_base", ctypes.c_int64),
                ("ring_pos", ctypes.c_int32), ("canon", ctypes.c_int8 * MAX_WORKERS),
                ("ring_rank", ctypes.c_int8 * MAX_WORKERS)]


class SesgdError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{lib().sesgd_strerror(code).decode()} ({code}){': ' + what if what else ''}")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u64, f32, f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_uint64, ctypes.c_float, ctypes.c_double)
        sig = {
            "sesgd_init": ([i32, i32, u64, ctypes.POINTER(P)], ctypes.c_int),
            "sesgd_destroy": ([P], None),
            "sesgd_groups": ([P, i64, P, P], ctypes.c_int),
            "sesgd_latency_model": ([i32, i32, f64, f64, f64, ctypes.POINTER(sesgd_cost)], ctypes.c_int),
            "sesgd_set_option": ([P, i32, i64], ctypes.c_int),
            "sesgd_attach": ([P, i32, i32, P], ctypes.c_int),
            "sesgd_register_bucket": ([P, i32, i64, P, P, P], ctypes.c_int),
            "sesgd_workspace_bytes": ([P, ctypes.POINTER(i64)], ctypes.c_int),
            "sesgd_workspace_prepare": ([P, P], ctypes.c_int),
            "sesgd_attach_peers": ([P, i32, i32, P, P], ctypes.c_int),
            "sesgd_begin_iter": ([P, i64], ctypes.c_int),
            "sesgd_begin_iter_device": ([P, i64, P], ctypes.c_int),
            "sesgd_device_iter_ptr": ([P, ctypes.POINTER(P)], ctypes.c_int),
            "sesgd_device_iter_read": ([P, ctypes.POINTER(sesgd_device_iter_state), P, i32], ctypes.c_int),
            "sesgd_sync_step": ([P, i32, f32, f32, P], ctypes.c_int),
            "sesgd_sync_step_host": ([P, i32, f32, f32, P, P, P], ctypes.c_int),
            "sesgd_sync_all": ([P, f32, f32, P], ctypes.c_int),
            "sesgd_global_average": ([P, i32, P, i32, P], ctypes.c_int),
            "sesgd_sync_all_host": ([P, f32, f32, P, P, P], ctypes.c_int),
            "sesgd_consensus": ([P, i32, P, i32, P, P], ctypes.c_int),
            "sesgd_set_weight_decay": ([P, f32], ctypes.c_int),
            "sesgd_attach_multicast": ([P, P], ctypes.c_int),
            "sesgd_pair_counts": ([P, i64, i64, P, P], ctypes.c_int),
            "sesgd_poll": ([P], ctypes.c_int),
            "sesgd_get_stats": ([P, i32, ctypes.POINTER(sesgd_stats)], ctypes.c_int),
            "sesgd_measure_hop": ([P, i32, i32, i32, P], ctypes.c_int),
            "sesgd_sync_all_pair": ([P, P, f32, f32, P], ctypes.c_int),
            "sesgd_launch_grid": ([P, ctypes.POINTER(i32)], ctypes.c_int),
            "sesgd_strerror": ([ctypes.c_int], ctypes.c_char_p),
            "sesgd_last_error": ([P], ctypes.c_char_p),
            "sesgd_probe_copy": ([P, P, i64, i32, P], ctypes.c_int),
            "sesgd_profile_read": ([P, P, i64, ctypes.POINTER(i32)], ctypes.c_int),
            "sesgd_probe_pingpong": ([P, P, i32, i32, u64, P, P], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc: int, ctx=None) -> None:
    if rc != OK:
        what = lib().sesgd_last_error(ctx).decode() if ctx else ""
        raise SesgdError(rc, what)


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


# ------------------------------------------------------------------ C-ABI calls
def sesgd_init(n: int, group_size: int, seed: int):
    ctx = ctypes.c_void_p()
    _check(lib().sesgd_init(n, group_size, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(ctx)))
    return ctx


def sesgd_destroy(ctx) -> None:
    lib().sesgd_destroy(ctx)


def sesgd_groups(ctx, it: int, n: int):
    perm = np.empty(n, np.int32)
    gof = np.empty(n, np.int32)
    _check(lib().sesgd_groups(ctx, it, perm.ctypes.data_as(ctypes.c_void_p),
                              gof.ctypes.data_as(ctypes.c_void_p)), ctx)
    return perm, gof


def sesgd_latency_model(n: int, group_size: int, nbytes: float, nu_Bps: float, tau_s: float) -> dict:
    out = sesgd_cost()
    _check(lib().sesgd_latency_model(n, group_size, float(nbytes), float(nu_Bps), float(tau_s),
                                     ctypes.byref(out)))
    return {f: getattr(out, f) for f, _ in sesgd_cost._fields_}


def sesgd_pair_counts(ctx, t0: int, T: int, counts_dev_ptr: int, stream: int = 0) -> None:
    """Accumulate into n*n device u64 counters how often each worker pair shares a group."""
    _check(lib().sesgd_pair_counts(ctx, t0, T, ctypes.c_void_p(int(counts_dev_ptr)),
                                   ctypes.c_void_p(int(stream))), ctx)


def sesgd_attach_multicast(ctx, mc_ptr: int) -> None:
    _check(lib().sesgd_attach_multicast(ctx, ctypes.c_void_p(int(mc_ptr))), ctx)


def sesgd_set_weight_decay(ctx, weight_decay: float) -> None:
    _check(lib().sesgd_set_weight_decay(ctx, float(weight_decay)), ctx)


def sesgd_set_option(ctx, option: int, value: int) -> None:
    _check(lib().sesgd_set_option(ctx, option, int(value)), ctx)


def sesgd_attach(ctx, device: int, local_workers) -> None:
    lw = np.ascontiguousarray(local_workers, np.int32)
    _check(lib().sesgd_attach(ctx, device, len(lw), lw.ctypes.data_as(ctypes.c_void_p)), ctx)


def sesgd_register_bucket(ctx, bucket: int, numel: int, x_ptrs, v_ptrs, g_ptrs) -> None:
    _check(lib().sesgd_register_bucket(ctx, bucket, numel, _ptr_array(x_ptrs), _ptr_array(v_ptrs),
                                       _ptr_array(g_ptrs)), ctx)


def sesgd_workspace_bytes(ctx) -> int:
    out = ctypes.c_int64()
    _check(lib().sesgd_workspace_bytes(ctx, ctypes.byref(out)), ctx)
    return out.value


def sesgd_workspace_prepare(ctx, local_ws_ptr: int) -> None:
    _check(lib().sesgd_workspace_prepare(ctx, ctypes.c_void_p(int(local_ws_ptr))), ctx)


def sesgd_attach_peers(ctx, n_ranks: int, rank: int, rank_ws_ptrs, worker_rank) -> None:
    wr = np.ascontiguousarray(worker_rank, np.int32)
    _check(lib().sesgd_attach_peers(ctx, n_ranks, rank, _ptr_array(rank_ws_ptrs),
                                    wr.ctypes.data_as(ctypes.c_void_p)), ctx)


def sesgd_begin_iter(ctx, it: int) -> None:
    _check(lib().sesgd_begin_iter(ctx, it), ctx)


def sesgd_begin_iter_device(ctx, it: int = ITER_NEXT, stream: int = 0) -> None:
    _check(lib().sesgd_begin_iter_device(ctx, it, stream), ctx)


def sesgd_device_iter_ptr(ctx) -> int:
    p = ctypes.c_void_p()
    _check(lib().sesgd_device_iter_ptr(ctx, ctypes.byref(p)), ctx)
    return int(p.value)


def sesgd_device_iter_read(ctx, n: int, m: int, nbuckets: int = 0) -> dict:
    st = sesgd_device_iter_state()
    calls = np.zeros(max(nbuckets, 1), np.int64)
    _check(lib().sesgd_device_iter_read(ctx, ctypes.byref(st), calls.ctypes.data_as(ctypes.c_void_p), nbuckets), ctx)
    return {"t": st.t, "seq": st.seq, "claim_base": st.claim_base, "ring_pos": st.ring_pos,
            "canon": list(st.canon[:n]), "ring_rank": list(st.ring_rank[:m]), "calls": calls[:nbuckets].tolist()}


def sesgd_sync_step(ctx, bucket: int, lr: float, momentum: float, stream: int = 0) -> None:
    _check(lib().sesgd_sync_step(ctx, bucket, lr, momentum, ctypes.c_void_p(int(stream))), ctx)


def sesgd_sync_all(ctx, lr: float, momentum: float, stream: int = 0) -> None:
    _check(lib().sesgd_sync_all(ctx, lr, momentum, ctypes.c_void_p(int(stream))), ctx)


def sesgd_sync_step_host(ctx, bucket: int, lr: float, momentum: float, g_host_ptrs, x_host_ptrs,
                         stream: int = 0) -> None:
    _check(lib().sesgd_sync_step_host(ctx, bucket, lr, momentum, _ptr_array(g_host_ptrs),
                                      _ptr_array(x_host_ptrs), ctypes.c_void_p(int(stream))), ctx)


def sesgd_sync_all_host(ctx, lr: float, momentum: float, g_host_ptrs, x_host_ptrs,
                        stream: int = 0) -> None:
    """g_host_ptrs / x_host_ptrs: flat [bucket * n_local + slot] host pointers."""
    _check(lib().sesgd_sync_all_host(ctx, lr, momentum, _ptr_array(g_host_ptrs),
                                     _ptr_array(x_host_ptrs), ctypes.c_void_p(int(stream))), ctx)


def sesgd_consensus(ctx, bucket: int, n: int, out_dev_ptr: int, row_ptrs=None, stream: int = 0) -> None:
    """Accumulates (sum of squared deviations, max abs deviation) into 2 device doubles."""
    rows = _ptr_array(row_ptrs) if row_ptrs is not None else None
    _check(lib().sesgd_consensus(ctx, bucket, rows, n, ctypes.c_void_p(int(out_dev_ptr)),
                                 ctypes.c_void_p(int(stream))), ctx)


def sesgd_global_average(ctx, bucket: int, n: int, row_ptrs=None, stream: int = 0) -> None:
    """row_ptrs: the n workers' device pointers (ascending worker id), or None (all local)."""
    rows = _ptr_array(row_ptrs) if row_ptrs is not None else None
    _check(lib().sesgd_global_average(ctx, bucket, rows, n, ctypes.c_void_p(int(stream))), ctx)


def sesgd_poll(ctx) -> None:
    _check(lib().sesgd_poll(ctx), ctx)


def sesgd_get_stats(ctx, bucket: int) -> dict:
    out = sesgd_stats()
    _check(lib().sesgd_get_stats(ctx, bucket, ctypes.byref(out)), ctx)
    return {f: getattr(out, f) for f, _ in sesgd_stats._fields_}


def sesgd_sync_all_pair(c0, c1, lr: float, momentum: float, stream: int = 0) -> None:
    _check(lib().sesgd_sync_all_pair(c0, c1, lr, momentum, ctypes.c_void_p(int(stream))), c0)


def sesgd_measure_hop(ctx, peer_rank: int, iters: int, initiator: bool, stream: int = 0) -> None:
    _check(lib().sesgd_measure_hop(ctx, peer_rank, iters, int(bool(initiator)), ctypes.c_void_p(int(stream))), ctx)


def sesgd_probe_copy(dst: int, src: int, nbytes: int, ctas: int, stream: int = 0) -> None:
    _check(lib().sesgd_probe_copy(ctypes.c_void_p(int(dst)), ctypes.c_void_p(int(src)), nbytes, ctas,
                                  ctypes.c_void_p(int(stream))))


def sesgd_probe_pingpong(my_flag: int, peer_flag: int, iters: int, initiator: bool, base: int,
                         out_ns_dev: int, stream: int = 0) -> None:
    _check(lib().sesgd_probe_pingpong(ctypes.c_void_p(int(my_flag)), ctypes.c_void_p(int(peer_flag)),
                                      iters, int(bool(initiator)), base,
                                      ctypes.c_void_p(int(out_ns_dev)), ctypes.c_void_p(int(stream))))


def sesgd_profile_read(ctx, grid: int):
    """-> (timers uint64[grid, 8], comm_ctas); see include/sesgd.h."""
    out = np.zeros((grid, 8), np.uint64)
    comm = ctypes.c_int32()
    _check(lib().sesgd_profile_read(ctx, out.ctypes.data_as(ctypes.c_void_p), out.size,
                                    ctypes.byref(comm)), ctx)
    return out, comm.value


def sesgd_launch_grid(ctx) -> int:
    out = ctypes.c_int32()
    _check(lib().sesgd_launch_grid(ctx, ctypes.byref(out)), ctx)
    return out.value

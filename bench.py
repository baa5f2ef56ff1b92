#!/usr/bin/env python
"""Benchmark of the SESGD group sync+update hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sesgd|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1]): n = 8 workers, group_size = 2, ResNet-50 DDP
buckets (5 buckets, 25,557,032 fp32 per worker), PARAM mode (Eq. 6), lr 0.1,
momentum 0.9.  N=1: all 8 workers resident on one B200 (kernel K6).  N>1: 8/N
workers per GPU, groups exchange over NVLink P2P (kernel K4 two-shot); the total work is
fixed ("scaling": "strong").  One step = one SESGD iteration over all buckets
of all workers (every row of SURVEY.md Sec. 8(a): schedule, local step, group
handshake + exchange + average, write-back).

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "group sync+update GB/s per GPU & iters/s at 1/2/4/8 B200 (fraction of roofline)"
N_WORKERS, GROUP_SIZE, LR, MU, SEED = 8, 2, 0.1, 0.9, 42
BYTES_PER_WORKER_ELEM = 20  # algorithmic HBM bytes: read g, v, x; write v, x (fp32)
NVLINK_PEER_GBS = 770.0     # measured peer copy per direction (B200_PROFILING.md), nominal 900
PAPER_CONTEXT = {"speedup_16w_0.1ms": 1.7, "speedup_16w_5ms": 5.0,
                 "source": "PAPER.md:7, P:411, P:436 (K80 + 1 Gbps Ethernet; end-to-end training, not this metric)"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="sesgd", choices=["sesgd", "reference"])
    p.add_argument("--workload", default="resnet50", choices=["resnet50", "vgg16", "config1"])
    p.add_argument("--workers", dest="n", type=int, default=N_WORKERS)  # (--n clashes with torchrun)
    p.add_argument("--group-size", type=int, default=GROUP_SIZE)
    p.add_argument("--mode", default="param", choices=["param", "grad"])
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--second-workload", type=int, default=1,
                   help="also time BASELINE cfg 3 (VGG-16, n=16, m=4) in the same run")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--p2p-variant", type=int, default=-1)
    p.add_argument("--discard", type=int, default=1)
    p.add_argument("--push-tma", type=int, default=0, help="two-shot: TMA bulk pushes (SESGD_OPT_PUSH_TMA)")
    p.add_argument("--release-delay", type=int, default=0, help="two-shot: SESGD_OPT_RELEASE_DELAY")
    p.add_argument("--release-every", type=int, default=0, help="two-shot: SESGD_OPT_RELEASE_EVERY")
    p.add_argument("--release-stagger", type=int, default=0, help="SESGD_OPT_RELEASE_STAGGER")
    p.add_argument("--payload-bf16", type=int, default=0, help="two-shot: bf16 reduce-scatter payload")
    p.add_argument("--path", default="auto", choices=["auto", "resident", "oneshot", "ring", "twoshot", "nvls"])
    p.add_argument("--fused", type=int, default=1, help="one-shot: one sesgd_sync_all launch per step")
    p.add_argument("--comm-batch", type=int, default=0)
    p.add_argument("--fold-lag", type=int, default=0)
    p.add_argument("--grid", type=int, default=0, help="CTAs per one-shot launch (0 = auto)")
    p.add_argument("--resident-unroll", type=int, default=0)
    p.add_argument("--protocol", type=int, default=-1, help="two-shot: SESGD_OPT_PROTOCOL (-1 auto)")
    p.add_argument("--ws-split", type=int, default=0, help="K4W-M: S warps (SESGD_OPT_WS_SPLIT, 0 = default)")
    p.add_argument("--hybrid", action="store_true", help="K6 for the all-local groups, then K4W-M (SESGD_OPT_WSM_HYBRID 1)")
    p.add_argument("--experiment", type=int, default=0,
                   help="SESGD_OPT_EXPERIMENT bits (measurement only: results are wrong)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(kernel: str, workload: str):
    """dram bytes per launch from the committed ncu --set full summary (profiles/traffic.json)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path)).get(f"{workload}/{kernel}")
    return None if d is None else d["bytes_per_launch"]


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    _NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
              0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
              0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def pcie_probe():
    """Measured pinned-host copy rates (tools/pcie_probe.py) committed under profiles/, or None."""
    path = os.path.join(ROOT, "profiles", "r01_pcie_probe_g1.json")
    return json.load(open(path)) if os.path.exists(path) else None


def local_groups_on_rank(perm, m, r, rank):
    """groups of the canonical partition `perm` whose m members all live on `rank` (worker w on
    rank w // r)"""
    return sum(1 for j in range(len(perm) // m) if all(int(w) // r == rank for w in perm[j * m:(j + 1) * m]))


def nvlink_algo_bytes(perm, m, r, world, L):
    """Algorithmic NVLink bytes of one iteration, per GPU per direction, max over GPUs.

    SURVEY.md Sec. 8(d) d2: a group spanning s GPUs costs each of them the bandwidth-optimal
    group-allreduce bound 2(s-1)/s * 4 B per element (co-resident members pre-combine; s = 1
    costs nothing).  perm = the iteration's canonical slots (group j = perm[j*m:(j+1)*m]),
    worker i lives on GPU i // r (r workers per GPU), L = elements per worker.
    """
    n = len(perm)
    per_gpu = [0.0] * world
    for j in range(n // m):
        ranks = {int(w) // r for w in perm[j * m:(j + 1) * m]}
        s_span = len(ranks)
        for rk in ranks:
            per_gpu[rk] += 2 * (s_span - 1) / s_span * 4 * L
    return max(per_gpu)


def workload_desc(workload, n, m, nb, L, mode):
    """The workload string both arms print in config.workload (same config, same metric)."""
    return (f"{cfg_label(workload, n, m)}: n={n} workers, group_size={m}, {workload} DDP buckets "
            f"({nb} buckets, {L:,} fp32 per worker), {mode.upper()} mode, lr {LR}, momentum {MU}")


def common_config(workload, n, m, mode):
    """config keys both arms print identically (same workload, same metric): the GPU arm's launch
    details (workers_per_gpu, path, ...) go to a separate "launch" object, the reference arm's
    coordinate sample to cpu_baseline.sample, so the two `config` objects are equal."""
    from paper_2007_00433_b200.workloads import WORKLOADS
    buckets = WORKLOADS[workload]
    return {"workload": workload_desc(workload, n, m, len(buckets), int(sum(buckets)), mode),
            "n": n, "group_size": m, "mode": mode}


def cfg_label(workload, n, m):
    """BASELINE.json config the run corresponds to (configs[1] = cfg2, configs[2] = cfg3)."""
    if workload == "resnet50" and n == 8 and m == 2:
        return "cfg2"
    if workload == "vgg16" and n == 16 and m == 4:
        return "cfg3"
    return "custom"


# ---------------------------------------------------------------- CPU oracle leg
def cpu_oracle_rate(n, m, budget_s, mode, L_total, workload):
    """Time the oracle as it stands (single-threaded C) on a bounded coordinate sample of the
    same workload (L_total fp32 per worker).  Returns (GB/s, sample description, seconds)."""
    import numpy as np

    import oracle
    import synth
    omode = oracle.MODE_PARAM if mode == "param" else oracle.MODE_GRAD

    def run(S, T, t0=0):
        coords = np.arange(S, dtype=np.int64) * 7 % L_total
        x = np.tile(synth.x0_host(S, coords=coords), (n, 1))
        v = np.zeros_like(x)
        t = time.perf_counter()
        oracle.run(n, m, SEED, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=omode, t0=t0, coords=coords)
        return time.perf_counter() - t

    probe_S, probe_T = 20000, 2
    dt = run(probe_S, probe_T)
    rate = n * probe_S * probe_T / dt  # worker-elements / s
    S = int(max(1000, min(L_total, rate * budget_s / (n * 4))))
    T = int(max(4, min(100, rate * budget_s / (n * S))))
    dt = run(S, T)
    gbs = BYTES_PER_WORKER_ELEM * n * S * T / dt / 1e9
    sample = (f"{workload}, n={n}, m={m}: {S} of {L_total:,} coordinates x {T} iterations "
              f"({n * S * T:.3g} worker-elements, {dt:.1f} s, single-threaded C oracle, fp32-emulate)")
    return gbs, sample, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth
    from paper_2007_00433_b200.workloads import WORKLOADS
    n, m = args.n, args.group_size
    L_total = int(sum(WORKLOADS[args.workload]))
    omode = oracle.MODE_PARAM if args.mode == "param" else oracle.MODE_GRAD
    # each step: one oracle iteration over a bounded coordinate sample of the workload
    steps, warm = args.steps, args.warmup
    per_step_budget = max(0.02, min(1.0, 120.0 / max(1, steps + warm)))
    S0 = 20000
    coords = np.arange(S0, dtype=np.int64)
    x = np.tile(synth.x0_host(S0, coords=coords), (n, 1))
    v = np.zeros_like(x)
    t = time.perf_counter()
    oracle.run(n, m, SEED, 1, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=omode, coords=coords)
    rate = n * S0 / (time.perf_counter() - t)
    S = int(max(1000, min(L_total, rate * per_step_budget / n)))
    coords = np.arange(S, dtype=np.int64)
    x = np.tile(synth.x0_host(S, coords=coords), (n, 1))
    v = np.zeros_like(x)
    for t in range(warm):
        oracle.run(n, m, SEED, 1, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=omode, t0=t, coords=coords)
    t0 = time.perf_counter()
    for t in range(warm, warm + steps):
        oracle.run(n, m, SEED, 1, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=omode, t0=t, coords=coords)
    dt = time.perf_counter() - t0
    gbs = BYTES_PER_WORKER_ELEM * n * S * steps / dt / 1e9
    sample = f"{args.workload}, n={n}, m={m}: {S} of {L_total:,} coordinates per step, 1 iteration per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**common_config(args.workload, n, m, args.mode),
                   "parallelism": f"sesgd groups over {args.gpus} GPU(s)"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU leg
def engine_options(args, C):
    return {k: v for k, v in ((C.OPT_COMM_BATCH, args.comm_batch), (C.OPT_FOLD_LAG, args.fold_lag),
                              (C.OPT_RESIDENT_UNROLL, args.resident_unroll), (C.OPT_PUSH_TMA, args.push_tma),
                              (C.OPT_RELEASE_DELAY, args.release_delay), (C.OPT_RELEASE_EVERY, args.release_every),
                              (C.OPT_RELEASE_STAGGER, args.release_stagger),
                              (C.OPT_PAYLOAD_BF16, args.payload_bf16), (C.OPT_EXPERIMENT, args.experiment),
                              (C.OPT_WS_SPLIT, args.ws_split),
                              ) if v} | {C.OPT_PROTOCOL: args.protocol} | ({C.OPT_WSM_HYBRID: 1} if args.hybrid else {})


class Dist:
    """rank / world / device plus the two collectives the timing needs (barrier, max over ranks)"""

    def __init__(self, world, local):
        import torch
        self.world, self.local = world, local
        self.dev = torch.device("cuda", local)

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max(self, v: float) -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


def measure(args, D, rank, workload, n, m, K, W, *, e2e_steps=0, clocks=None):
    """Time K SESGD iterations (after W warm-up ones) of `workload` with n workers, group size m,
    n / world per GPU; returns the per-workload fields of the JSON line (value, roofline, ...)."""
    import numpy as np
    import torch

    import synth
    from paper_2007_00433_b200 import sesgd as C
    from paper_2007_00433_b200.engine import SESGDEngine
    from paper_2007_00433_b200.workloads import WORKLOADS

    world = D.world
    if n % world:
        raise SystemExit("n must be a multiple of the GPU count")
    buckets = list(WORKLOADS[workload])
    L = sum(buckets)
    mode = C.MODE_PARAM_AVG if args.mode == "param" else C.MODE_GRAD_AVG
    path = {"auto": C.PATH_AUTO, "resident": C.PATH_RESIDENT, "oneshot": C.PATH_ONESHOT,
            "ring": C.PATH_RING, "twoshot": C.PATH_TWOSHOT, "nvls": C.PATH_NVLS}[args.path]
    eng = SESGDEngine(n, m, buckets, seed=SEED, mode=mode, rank=rank, world=world,
                      p2p_variant=args.p2p_variant, discard=args.discard, grid=args.grid,
                      options=engine_options(args, C), path=path)
    r = eng.r
    stream = torch.cuda.current_stream(D.dev)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for s, w in enumerate(eng.local_workers):
        for b, Lb in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), Lb, int(offs[b]), stream.cuda_stream)
            synth.fill_grad_device(eng.g(s, b).data_ptr(), Lb, int(offs[b]), w, 0, stream.cuda_stream)
    torch.cuda.synchronize()
    nb = len(buckets)
    fused = bool(args.fused)  # one sesgd_sync_all launch per step (all buckets)
    launches_per_step = 1 if fused else nb  # event pairs per step
    kernels_per_step = nb if args.path == "ring" else launches_per_step  # K5 launches per bucket
    t_next = 0
    for _ in range(W):
        eng.step(t_next, LR, MU, stream, fused=fused)
        t_next += 1
    eng.poll()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(launches_per_step)] for _ in range(K)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    with (clocks if clocks is not None else ClockSampler(D.local)) as clk:
        start.record(stream)
        for k in range(K):
            eng.begin_iter(t_next)
            if fused:
                ev[k][0][0].record(stream)
                eng.sync_all(LR, MU, stream)
                ev[k][0][1].record(stream)
            else:
                for b in range(nb):
                    ev[k][b][0].record(stream)
                    eng.sync_step(b, LR, MU, stream)
                    ev[k][b][1].record(stream)
            t_next += 1
        end.record(stream)
        D.barrier()
    eng.poll()
    ms_total = D.max(start.elapsed_time(end))
    ms_step = ms_total / K
    launch_ms = [[e0.elapsed_time(e1) for (e0, e1) in ev[k]] for k in range(K)]
    kern_ms_total = D.max(sum(map(sum, launch_ms)))
    # per-step kernel time distribution (median and p90), max over ranks
    step_ms = sorted(sum(row) for row in launch_ms)
    kern_p50 = D.max(step_ms[(K - 1) // 2])
    kern_p90 = D.max(step_ms[min(K - 1, int(0.9 * K))])
    total_bytes = BYTES_PER_WORKER_ELEM * L * n  # whole job, per step
    value = total_bytes / (ms_step * 1e-3) / 1e9
    hbm_peak, peak_src = measured_peaks()
    algo_bytes_per_step_gpu = BYTES_PER_WORKER_ELEM * L * r
    resident = (world == 1 and args.path in ("auto", "resident"))
    # the path AUTO resolves to (sesgd_capi.cu resolve_path): K4 two-shot unless COMM CTAs
    eff_path = args.path
    if eff_path == "auto" and not resident:
        eff_path = "oneshot" if args.p2p_variant >= 1 else "twoshot"
    if resident:
        kernel = "k6_resident"
        achieved = algo_bytes_per_step_gpu * K / (kern_ms_total * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "peak_source": peak_src,
                "algo_bytes_per_launch": ([BYTES_PER_WORKER_ELEM * L * r] if fused else
                                          [BYTES_PER_WORKER_ELEM * Lb * r for Lb in buckets]),
                "kernel": kernel}
    else:
        proto = args.protocol if args.protocol >= 0 else (2 if r <= 8 else 1)  # auto (sesgd_capi.cu)
        if args.push_tma or args.payload_bf16:
            proto = 0 if args.protocol < 0 else proto
        # several workers per GPU; --hybrid: K6 updates the all-local groups first, then K4W-M
        # (SESGD_OPT_WSM_HYBRID); the per-launch events cover both kernels
        k4w = "k4w_twoshot" if r == 1 else ("k6_resident+k4w_multi" if args.hybrid else "k4w_multi")
        kernel = {"twoshot": k4w if proto == 2 else "k4_twoshot",
                  "ring": "k5_ring", "nvls": "k4_nvls"}.get(eff_path, "k3_push")
        # NVLink: bandwidth-optimal group-allreduce bytes per GPU per direction, from the
        # actual schedule of the timed iterations: a group spanning s GPUs costs every one
        # of them 2(s-1)/s * 4 B per element (co-resident members pre-combine); max over
        # GPUs, mean over the timed iterations.
        nvl_steps = [nvlink_algo_bytes(eng.groups(t)[0], m, r, world, L) for t in range(t_next - K, t_next)]
        nvl_bytes = sum(nvl_steps) / len(nvl_steps)
        achieved_nvl = nvl_bytes * K / (kern_ms_total * 1e-3) / 1e9
        achieved_hbm = algo_bytes_per_step_gpu * K / (kern_ms_total * 1e-3) / 1e9
        t_hbm = algo_bytes_per_step_gpu / (hbm_peak * 1e9)
        t_nvl = nvl_bytes / (NVLINK_PEER_GBS * 1e9)
        if t_nvl >= t_hbm and nvl_bytes > 0:
            roof = {"bound": "nvlink", "achieved": achieved_nvl, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                    "frac": achieved_nvl / NVLINK_PEER_GBS,
                    "peak_source": "measured peer copy per direction, B200_PROFILING.md (nominal 900)"}
        else:
            roof = {"bound": "hbm", "achieved": achieved_hbm, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved_hbm / hbm_peak, "peak_source": peak_src}
        roof.update({"hbm_achieved": achieved_hbm, "nvlink_algo_bytes_per_step": nvl_bytes,
                     "t_roof_us": max(t_hbm, t_nvl) * 1e6, "kernel": kernel})
    roof["traffic"] = traffic_for(kernel, f"{workload}_n{n}_m{m}_g{world}")
    if kernel == "k6_resident+k4w_multi":  # the K6 launch happens only in iterations with an all-local group
        extra_k6 = sum(1 for t in range(t_next - K, t_next) if local_groups_on_rank(eng.groups(t)[0], m, r, rank) > 0)
        gpu_launches_extra = extra_k6
    else:
        gpu_launches_extra = 0

    # ---- e2e through the C-ABI host-buffer call (H2D of g, D2H of x inside the timed region)
    e2e = None
    if e2e_steps > 0:
        g_host = [[torch.empty(Lb, dtype=torch.float32).pin_memory() for _ in range(r)] for Lb in buckets]
        x_host = [[torch.empty(Lb, dtype=torch.float32).pin_memory() for _ in range(r)] for Lb in buckets]
        for b in range(nb):
            for s in range(r):
                g_host[b][s].copy_(eng.g(s, b))
        eng.step_host(t_next, LR, MU, g_host, x_host, stream)
        t_next += 1
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            eng.step_host(t_next, LR, MU, g_host, x_host, stream)
            t_next += 1
        e1.record(stream)
        D.barrier()
        e2e_ms = D.max(e0.elapsed_time(e1)) / e2e_steps
        e2e = {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 4 * L * n, "d2h_bytes_per_step": 4 * L * n,
               "ms_per_step": e2e_ms, "steps": e2e_steps,
               "api": "sesgd_sync_all_host (pinned host g in, updated x out, every worker; H2D / "
                      "kernels / D2H of different buckets pipelined on copy streams)"}
        probe = pcie_probe()
        if probe is not None:  # the e2e step against its own bound: both copy directions at once
            bound_ms = 4 * L * r / (probe["both_gbs_per_dir"] * 1e6)
            e2e["pcie_bound"] = {"ms_per_step": bound_ms, "frac": bound_ms / e2e_ms,
                                 "gbs_per_dir": probe["both_gbs_per_dir"],
                                 "source": "tools/pcie_probe.py, profiles/r01_pcie_probe_g1.json "
                                           "(pinned H2D and D2H of the same bytes concurrently)"}
    eng.poll()
    stats = [eng.stats(b) for b in range(nb)]
    # consistency of the workers' parameters after the run (K9), outside the timed region
    css, cmx = eng.consensus(stream)
    out = {
        "config": {**common_config(workload, n, m, args.mode),
                   "parallelism": f"sesgd groups over {world} GPU(s)"},
        "launch": {"workers_per_gpu": r,
                   "path": "resident (K6)" if resident else {
                       "twoshot": "two-shot reduce-scatter/all-gather push over NVLink P2P ("
                                  + {"k4w_twoshot": "K4W, warp-specialised", "k4w_multi": "K4W-M, warp-specialised,"
                                     " several workers per GPU"}.get(kernel, "K4") + ")",
                       "ring": "ring inside each group over NVLink P2P (K5)"}.get(
                           eff_path, "one-shot push over NVLink P2P (K3)"),
                   "l2": f"inputs larger than L2: {3 * 4 * L * r / 1e9:.2f} GB working set per GPU vs 126 MB L2; no flush"},
        "value": value, "ms_per_step": ms_step, "steps": K, "warmup": W,
        "iters_per_s": 1e3 / ms_step, "gbs_per_gpu": value / world,
        "kernel_ms_per_step": {"p50": kern_p50, "p90": kern_p90},
        "roofline": roof, "e2e": e2e, "gpu_launches": K * kernels_per_step + gpu_launches_extra,
        "kernel_rounds_per_bucket": stats[0]["handshake_rounds"],
        "consistency": {"after_iterations": t_next, "sum_sq_dev_from_mean": css,
                        "rms_dev": (css / (n * L)) ** 0.5, "max_abs_dev": cmx,
                        "note": "SESGD keeps the workers consistent (P:430-433); x0 ~ U[-1/8, 1/8)"},
        "clocks": clk.summary() if clocks is None else None,
        "L": L, "nb": nb,
    }
    eng.close()
    del eng
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def measure_tau(D, rank):
    """Per-hop handshake latency t_tau (Eq. 2) in this run: K7 flag ping-pong between
    rank 0 and rank 1 over NVLink (N >= 2; symmetric-memory flags), or between two concurrent
    kernels on this GPU through L2 (N = 1: no NVLink on the path, the on-chip lower bound)."""
    import torch
    from paper_2007_00433_b200 import sesgd as C
    iters = 5000
    out_ns = torch.zeros(1, dtype=torch.int64, device=D.dev)
    if D.world == 1:
        flags = torch.zeros(64, dtype=torch.int64, device=D.dev)
        s1, s2 = torch.cuda.Stream(D.dev), torch.cuda.Stream(D.dev)
        dummy = torch.zeros(1, dtype=torch.int64, device=D.dev)
        base = 1
        for _ in range(2):
            C.sesgd_probe_pingpong(flags.data_ptr(), flags.data_ptr() + 256, iters, True, base,
                                   out_ns.data_ptr(), s1.cuda_stream)
            C.sesgd_probe_pingpong(flags.data_ptr() + 256, flags.data_ptr(), iters, False, base,
                                   dummy.data_ptr(), s2.cuda_stream)
            base += 2 * iters + 2
            torch.cuda.synchronize()
        ns = int(out_ns.item())
        return {"tau_us": ns / iters / 2 / 1e3, "scope": "intra-GPU (two concurrent kernels, flags in L2; "
                "N = 1 has no NVLink hop)", "iters": iters}
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    buf = symm_mem.empty(64, dtype=torch.int64, device=D.dev)
    buf.zero_()
    hdl = symm_mem.rendezvous(buf, dist.group.WORLD)
    D.barrier()
    if rank < 2:
        other = 1 - rank
        base = 1
        for _ in range(2):
            C.sesgd_probe_pingpong(hdl.buffer_ptrs[rank], hdl.buffer_ptrs[other], iters, rank == 0, base,
                                   out_ns.data_ptr(), torch.cuda.current_stream(D.dev).cuda_stream)
            base += 2 * iters + 2
            torch.cuda.synchronize()
    D.barrier()
    ns = D.max(float(out_ns.item()) if rank == 0 else 0.0)
    return {"tau_us": ns / iters / 2 / 1e3, "scope": "NVLink (rank 0 <-> rank 1 through NVSwitch)",
            "iters": iters}


def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"nproc": usable, "cpu_count": os.cpu_count(), "cpu_model": model}


def _oracle_slice(args):
    """one process of the all-core oracle leg: the unchanged single-threaded oracle on its own
    disjoint coordinate subset (coordinates are independent); returns its compute seconds"""
    n, m, mode, S, T, part, parts, L_total, q, bar = args
    import numpy as np

    import oracle
    import synth
    omode = oracle.MODE_PARAM if mode == "param" else oracle.MODE_GRAD
    coords = (np.arange(part, S * parts, parts, dtype=np.int64) * 7) % L_total
    x = np.tile(synth.x0_host(len(coords), coords=coords), (n, 1))
    v = np.zeros_like(x)
    bar.wait()
    t = time.perf_counter()
    oracle.run(n, m, SEED, T, x, v, s_g=synth.SEED_G, lr=LR, mu=MU, mode=omode, coords=coords)
    q.put(time.perf_counter() - t)


def cpu_oracle_all_cores(n, m, mode, L_total, workload, rate_1core, budget_s):
    """P = usable cores processes, each the plain oracle on 1/P of a coordinate sample; the
    aggregate is total worker-elements / the slowest process's compute time"""
    import multiprocessing as mp
    P = cpu_info()["nproc"] or 1
    S = int(max(1000, min(L_total, rate_1core * P * budget_s / (n * 4))))
    T = 4
    ctx = mp.get_context("spawn")
    q, bar = ctx.Queue(), ctx.Barrier(P)
    procs = [ctx.Process(target=_oracle_slice, args=((n, m, mode, S // P, T, i, P, L_total, q, bar),))
             for i in range(P)]
    for pr in procs:
        pr.start()
    secs = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    dt = max(secs)
    gbs = BYTES_PER_WORKER_ELEM * n * (S // P) * P * T / dt / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": P, "kind": "oracle",
            "sample": (f"{workload}, n={n}, m={m}: {P} processes x {S // P} coordinates x {T} iterations, "
                       f"each the unchanged single-threaded oracle on a disjoint coordinate subset; "
                       f"slowest process {dt:.1f} s")}


def run_sesgd(args):
    import torch
    import torch.distributed as dist

    from paper_2007_00433_b200 import sesgd as C

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    n, m = args.n, args.group_size
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    D = Dist(world, local)
    K, W = args.steps, args.warmup
    main = measure(args, D, rank, args.workload, n, m, K, W, e2e_steps=args.e2e_steps)
    L, nb = main.pop("L"), main.pop("nb")
    # BASELINE configs[2] (VGG-16, n = 16, group_size 4) in the same run, as the north star asks
    second = None
    if args.second_workload and args.workload == "resnet50" and (n, m) == (8, 2):
        second = measure(args, D, rank, "vgg16", 16, 4, max(3, min(K, 20)), max(3, min(W, 5)))
        for k in ("L", "nb", "e2e"):
            second.pop(k, None)
    tau = measure_tau(D, rank)
    lat = C.sesgd_latency_model(n, m, 4.0 * L / nb, NVLINK_PEER_GBS * 1e9, tau["tau_us"] * 1e-6)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gbs, sample, dt = cpu_oracle_rate(n, m, args.cpu_seconds, args.mode, L, args.workload)
        cpu = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample, **cpu_info()}
        rate_1core = gbs * 1e9 / BYTES_PER_WORKER_ELEM  # worker-elements / s
        try:
            cpu["all_cores"] = cpu_oracle_all_cores(n, m, args.mode, L, args.workload, rate_1core,
                                                    args.cpu_seconds)
        except Exception as e:  # reported, never fatal: the GPU line stands on its own
            cpu["all_cores"] = {"error": repr(e)}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": main["value"], "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": main["config"],
            "launch": main["launch"],
            "iters_per_s": main["iters_per_s"],
            "gbs_per_gpu": main["gbs_per_gpu"],
            "kernel_ms_per_step": main["kernel_ms_per_step"],
            "roofline": main["roofline"],
            "cpu_baseline": cpu,
            "e2e": main["e2e"],
            "gpu_launches": main["gpu_launches"],
            "clocks": main["clocks"],
            "handshakes": {
                "sesgd_per_tensor": lat["sesgd_handshakes"], "ring_per_tensor": lat["ring_handshakes"],
                "kernel_rounds_per_bucket": main["kernel_rounds_per_bucket"],
                "tau_measured": tau,
                "model": (f"Eq.2/Eq.3 exact (sesgd_latency_model), nu={NVLINK_PEER_GBS:.0f} GB/s, "
                          f"tau={tau['tau_us']:.2f} us measured in this run (K7 flag ping-pong)"),
                "model_ratio": lat["ratio"],
            },
            "paper_context": PAPER_CONTEXT,
            "consistency": main["consistency"],
            "workloads": {"cfg3_vgg16": second} if second is not None else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_sesgd(args)


if __name__ == "__main__":
    sys.exit(main())

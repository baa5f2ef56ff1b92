"""Per-rank body of the multi-GPU parity test (launched by tests/test_gpu_multigpu.py via
torch.distributed.run, one process per GPU), or -- with --loopback R -- all R virtual ranks in
ONE process on ONE GPU (engine.LoopbackGroup: the same kernels, flags and workspaces, peers in
local memory).  Runs T SESGD iterations through the multi-GPU paths and saves every rank's
workers' x and v for the parent to compare with the oracle."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import SESGDEngine  # noqa: E402


def _options(a):
    return {k: v for k, v in ((C.OPT_COMM_BATCH, a.batch), (C.OPT_FOLD_LAG, a.lag),
                              (C.OPT_PUSH_TMA, a.tma), (C.OPT_LOCAL_PERIOD, a.period),
                              (C.OPT_SCHEDULE, a.schedule), (C.OPT_PAYLOAD_BF16, a.bf16),
                              (C.OPT_RELEASE_EVERY, a.release_every), (C.OPT_WSM_HYBRID, a.hybrid)) if v} | {
        C.OPT_PROTOCOL: a.protocol}


def _padded(idx, buckets, offsets):
    """global (unpadded) element indices -> the engine's aligned flat layout"""
    starts = torch.tensor(np.concatenate([[0], np.cumsum(buckets)[:-1]]), device=idx.device)
    b = torch.searchsorted(starts, idx, right=True) - 1
    return idx - starts[b] + torch.tensor(offsets, device=idx.device)[b]


def _rows(eng, flat, buckets, coords):
    if coords is None:
        return np.stack([torch.cat([eng.view(f, b) for b in range(len(buckets))]).cpu().numpy() for f in flat])
    idx = _padded(torch.from_numpy(coords).to(eng.device), buckets, eng.offsets)
    return np.stack([f[idx].cpu().numpy() for f in flat])


def run_iterations(engs, a, buckets, offs, host_step):
    """T iterations from t0.  --devit 0: host iterations (begin_iter + sync per iteration);
    1: device iteration state, eager (sesgd_begin_iter_device + gradient fill reading the device's
    t + sync, enqueued per iteration); 2: the same iteration captured ONCE as a CUDA graph and
    replayed T times; 3: T/3 host iterations, the graph, then host iterations again (the state
    moves host -> device -> host)."""
    t0, T = a.t0, a.iters
    if a.devit == 0:
        for t in range(t0, t0 + T):
            host_step(t)
        return
    h = T // 3 if a.devit == 3 else 0
    for t in range(t0, t0 + h):
        host_step(t)
    for e in engs:
        e.set_device_iter(True)
    if h == 0 and t0 > 0:  # so that the first ITER_NEXT lands on t0
        for e in engs:
            e.begin_iter_device(t0 - 1)

    def produce(e, s):
        tp = e.t_device_ptr()
        for slot, w in enumerate(e.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_grad_device_at(e.g(slot, b).data_ptr(), L, int(offs[b]), w, tp, s.cuda_stream)

    nd = T - 2 * h
    if a.devit == 1:
        for _ in range(nd):
            for e in engs:
                e.enqueue_iteration(0.1, 0.9, produce, bool(a.fused))
    else:
        graphs = [e.capture_iteration(0.1, 0.9, produce, bool(a.fused)) for e in engs]
        for _ in range(nd):
            for e, g in zip(engs, graphs):
                e.replay_iteration(g)
    if a.devit == 3:
        for e in engs:
            e.set_device_iter(False)
        for t in range(t0 + h + nd, t0 + T):
            host_step(t)


def loopback(a):
    """R virtual ranks on cuda:0 (SESGD_OPT_SM_BUDGET = SMs / R each, one stream each)"""
    from paper_2007_00433_b200.engine import LoopbackGroup
    torch.cuda.set_device(0)
    buckets = [int(b) for b in a.buckets.split(",")]
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    coords = np.load(a.coords) if a.coords else None
    grp = LoopbackGroup(a.loopback, a.workers, a.gsize, buckets, seed=42, mode=a.mode, grid=a.grid,
                        timeout_ms=10000, p2p_variant=a.variant, path=a.path, hop_delay_ns=a.hop_ns,
                        weight_decay=a.wd, options=_options(a))
    for eng in grp:
        st = eng.stream.cuda_stream
        for s in range(eng.r):
            for b, L in enumerate(buckets):
                synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), st)
    def host_step(t):
        for eng in grp:
            st = eng.stream.cuda_stream
            for s, w in enumerate(eng.local_workers):
                for b, L in enumerate(buckets):
                    synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, t, st)
        grp.step(t, 0.1, 0.9, fused=bool(a.fused))

    run_iterations(list(grp), a, buckets, offs, host_step)
    if a.final_avg:
        grp.global_average()
    grp.synchronize()
    grp.poll()
    cons = np.array(grp.consensus() if a.consensus else (0.0, 0.0))
    for eng in grp:
        stats = eng.stats(0)
        np.savez(f"{a.out}.rank{eng.rank}.npz", X=_rows(eng, eng.x_flat, buckets, coords),
                 V=_rows(eng, eng.v_flat, buckets, coords), workers=np.array(eng.local_workers),
                 flag_messages=stats["flag_messages"], payload=stats["payload_bytes_in"], cons=cons)
    grp.close()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workers", type=int, required=True)
    p.add_argument("--gsize", type=int, required=True)
    p.add_argument("--iters", type=int, required=True)
    p.add_argument("--buckets", required=True)
    p.add_argument("--mode", type=int, default=0)
    p.add_argument("--t0", type=int, default=0)
    p.add_argument("--grid", type=int, default=0)
    p.add_argument("--variant", type=int, default=-1)
    p.add_argument("--fused", type=int, default=1)
    p.add_argument("--path", type=int, default=0)
    p.add_argument("--hop-ns", type=int, default=0)
    p.add_argument("--batch", type=int, default=0)
    p.add_argument("--lag", type=int, default=0)
    p.add_argument("--tma", type=int, default=0)
    p.add_argument("--period", type=int, default=1)
    p.add_argument("--final-avg", type=int, default=0)
    p.add_argument("--schedule", type=int, default=0)
    p.add_argument("--consensus", type=int, default=0)
    p.add_argument("--wd", type=float, default=0.0)
    p.add_argument("--bf16", type=int, default=0)
    p.add_argument("--protocol", type=int, default=-1)  # SESGD_OPT_PROTOCOL, -1 = auto
    p.add_argument("--release-every", type=int, default=0)
    p.add_argument("--loopback", type=int, default=0)
    p.add_argument("--devit", type=int, default=0)  # device iteration state: 1 eager, 2 graph, 3 mixed
    p.add_argument("--hybrid", type=int, default=0)  # SESGD_OPT_WSM_HYBRID
    p.add_argument("--coords", default="")
    p.add_argument("--out", required=True)
    a = p.parse_args()
    if a.loopback:
        return loopback(a)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    buckets = [int(b) for b in a.buckets.split(",")]
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    eng = SESGDEngine(a.workers, a.gsize, buckets, seed=42, mode=a.mode, rank=rank, world=world,
                      grid=a.grid, timeout_ms=10000, p2p_variant=a.variant, path=a.path,
                      hop_delay_ns=a.hop_ns, weight_decay=a.wd,
                      options=_options(a))
    st = torch.cuda.current_stream().cuda_stream
    for s in range(eng.r):
        for b, L in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), st)
    def host_step(t):
        for s, w in enumerate(eng.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, t, st)
        eng.step(t, 0.1, 0.9, fused=bool(a.fused))

    run_iterations([eng], a, buckets, offs, host_step)
    if a.final_avg:
        eng.global_average()
    torch.cuda.synchronize()
    eng.poll()
    coords = np.load(a.coords) if a.coords else None
    X = _rows(eng, eng.x_flat, buckets, coords)
    V = _rows(eng, eng.v_flat, buckets, coords)
    stats = eng.stats(0)
    cons = np.array(eng.consensus() if a.consensus else (0.0, 0.0))
    np.savez(f"{a.out}.rank{rank}.npz", X=X, V=V, workers=np.array(eng.local_workers),
             flag_messages=stats["flag_messages"], payload=stats["payload_bytes_in"], cons=cons)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

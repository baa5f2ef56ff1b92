#!/usr/bin/env python
"""Per-CTA phase timers of the one-shot K3 / two-shot K4 kernels (SESGD_OPT_PROFILE), multi-GPU.

    python -m torch.distributed.run --nproc-per-node 2 tools/k3_phase_profile.py --workers 2

Runs the cfg-2 ResNet-50 buckets, then prints, per rank, the mean per-launch time COMM CTAs
spend waiting for staged chunks / pushing / releasing flags and COMPUTE CTAs spend staging /
folding (ns from %globaltimer).  Diagnostic only (timers perturb the kernel slightly).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import SESGDEngine  # noqa: E402
from paper_2007_00433_b200.workloads import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--gsize", type=int, default=2)
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--lag", type=int, default=0)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--path", type=int, default=0, help="SESGD_PATH_* (4 = two-shot)")
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--rel-delay", type=int, default=0)
    ap.add_argument("--rel-every", type=int, default=0)
    ap.add_argument("--protocol", type=int, default=0)
    ap.add_argument("--ws-split", type=int, default=0)
    ap.add_argument("--experiment", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/k3_phases.json")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    buckets = list(WORKLOADS["resnet50"])
    opts = {}
    if a.batch:
        opts[C.OPT_COMM_BATCH] = a.batch
    if a.lag:
        opts[C.OPT_FOLD_LAG] = a.lag
    if a.rel_delay:
        opts[C.OPT_RELEASE_DELAY] = a.rel_delay
    if a.rel_every:
        opts[C.OPT_RELEASE_EVERY] = a.rel_every
    if a.protocol:
        opts[C.OPT_PROTOCOL] = a.protocol
    if a.ws_split:
        opts[C.OPT_WS_SPLIT] = a.ws_split
    if a.experiment:
        opts[C.OPT_EXPERIMENT] = a.experiment
    eng = SESGDEngine(a.workers, a.gsize, buckets, rank=rank, world=world, p2p_variant=a.variant,
                      path=a.path, grid=a.grid, options=opts)
    C.sesgd_set_option(eng.ctx, C.OPT_PROFILE, 1)
    st = torch.cuda.current_stream()
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for s, w in enumerate(eng.local_workers):
        for b, L in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), st.cuda_stream)
            synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, 0, st.cuda_stream)
    for t in range(3):
        eng.step(t, 0.1, 0.9, fused=bool(a.fused))
    torch.cuda.synchronize()
    grid = C.sesgd_launch_grid(eng.ctx)
    C.sesgd_profile_read(eng.ctx, grid)  # reset
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(3, 3 + a.iters):
        eng.step(t, 0.1, 0.9, fused=bool(a.fused))
    e1.record()
    torch.cuda.synchronize()
    prof, comm = C.sesgd_profile_read(eng.ctx, grid)
    launches = a.iters * len(buckets)
    cm, cp = prof[:comm].astype(np.float64), prof[comm:].astype(np.float64)
    res = {"rank": rank, "grid": grid, "comm_ctas": comm, "ms_per_iter": e0.elapsed_time(e1) / a.iters,
           "per_iter_us": {
               "comm_wait_staged": cm[:, 0].mean() / a.iters / 1e3,
               "comm_push": cm[:, 1].mean() / a.iters / 1e3,
               "comm_release": cm[:, 2].mean() / a.iters / 1e3,
               "comm_total": cm[:, 3].mean() / a.iters / 1e3,
               "compute_stage": cp[:, 0].mean() / a.iters / 1e3,
               "compute_fold": cp[:, 1].mean() / a.iters / 1e3,  # two-shot: reduce
               "compute_finish": cp[:, 3].mean() / a.iters / 1e3,  # two-shot only
               "compute_release": cp[:, 4].mean() / a.iters / 1e3,  # two-shot only
               "compute_total": cp[:, 2].mean() / a.iters / 1e3,
               "compute_total_max": cp[:, 2].max() / a.iters / 1e3},
           "launches_seen": int(prof[:, 7].max()), "launches": launches}
    if a.protocol == 2:  # K4W warp groups (p2p_ws.cu): leader-thread timers per CTA
        us = lambda col: cp[:, col].mean() / a.iters / 1e3  # noqa: E731
        res["per_iter_us"] = {"S_stream": us(0), "S_wait_ring_free": us(4), "R_fold": us(1),
                              "R_wait_ring_full": us(5), "R_poll_spin": us(6), "F_gather": us(3),
                              "F_poll_spin": us(2), "S_stream_max": cp[:, 0].max() / a.iters / 1e3,
                              "F_gather_max": cp[:, 3].max() / a.iters / 1e3}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps(allres, indent=1))
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(allres, open(a.out, "w"), indent=1)
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

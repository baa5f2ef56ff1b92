#!/usr/bin/env python
"""NCCL baselines for the SESGD hot path (one worker per GPU; run under torch.distributed.run).

    python -m torch.distributed.run --nproc-per-node 4 tools/nccl_baseline.py --out gpurun_out/nccl.json

Same workload as bench.py (ResNet-50 DDP buckets, lr 0.1, momentum 0.9, n = world), timed
with CUDA events (max over ranks, median of --iters):
  * ring_sgd  -- Eq. 4: per bucket NCCL all_reduce(AVG) of the gradient over
                 all n workers, then torch momentum SGD (v = mu v + g; x -= lr v);
  * sesgd_nccl -- Eq. 6 with stock NCCL: x_hat = x - lr (mu v + g) with torch ops, then
                 all_reduce(AVG) of x_hat inside the iteration's shuffle-exchange groups
                 through cached per-group sub-communicators (dist.new_group);
  * sesgd_libsesgd -- the same iteration through libsesgd's fused one-shot kernel.
These are BASELINES (stock library calls), not the product.
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import SESGDEngine  # noqa: E402
from paper_2007_00433_b200.workloads import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gsize", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--out", default="gpurun_out/nccl_baseline.json")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    n, m = world, a.gsize
    buckets = list(WORKLOADS[a.workload])
    L = sum(buckets)
    lr, mu = 0.1, 0.9
    xs = [torch.randn(b, device=dev) * 0.1 for b in buckets]
    vs = [torch.zeros(b, device=dev) for b in buckets]
    gs = [torch.randn(b, device=dev) * 0.01 for b in buckets]
    stream = torch.cuda.current_stream()
    ctx = C.sesgd_init(n, m, 42)  # schedule only (same partitions as libsesgd)
    groups_cache = {}

    def group_of(t):
        perm, gof = C.sesgd_groups(ctx, t, n)
        j = int(gof[rank])
        members = tuple(int(w) for w in perm[j * m:(j + 1) * m])
        key = tuple(tuple(int(w) for w in perm[q * m:(q + 1) * m]) for q in range(n // m))
        if key not in groups_cache:  # every rank creates every group of the partition (collective)
            groups_cache[key] = {g: dist.new_group(list(g)) for g in key}
        return groups_cache[key][members]

    def ring_sgd(t):
        for x, v, g in zip(xs, vs, gs):
            gg = g.clone()
            dist.all_reduce(gg, op=dist.ReduceOp.AVG)
            v.mul_(mu).add_(gg)
            x.add_(v, alpha=-lr)

    def sesgd_nccl(t):
        pg = group_of(t)
        for x, v, g in zip(xs, vs, gs):
            v.mul_(mu).add_(g)
            x.add_(v, alpha=-lr)  # x_hat
            dist.all_reduce(x, op=dist.ReduceOp.AVG, group=pg)

    eng = SESGDEngine(n, m, buckets, rank=rank, world=world)

    def sesgd_lib(t):
        eng.step(t, lr, mu, stream)

    res = {"n": n, "m": m, "workload": a.workload, "elements_per_worker": L}
    for name, fn in (("ring_sgd", ring_sgd), ("sesgd_nccl", sesgd_nccl), ("sesgd_libsesgd", sesgd_lib)):
        for t in range(3):  # warm-up (also creates the sub-communicators of the first partitions)
            fn(t)
        torch.cuda.synchronize()
        dist.barrier()
        # pre-create the sub-communicators of the timed iterations outside the timed region
        if name == "sesgd_nccl":
            for t in range(100, 100 + a.iters):
                group_of(t)
        times = []
        for t in range(100, 100 + a.iters):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(t)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        res[name] = {"ms_per_iter": ms, "algo_gbs_per_gpu": 20 * L / (ms * 1e-3) / 1e9}
    eng.close()
    C.sesgd_destroy(ctx)
    if rank == 0:
        print(json.dumps(res, indent=1))
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

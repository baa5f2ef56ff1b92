#!/usr/bin/env python
"""BASELINE config 4: group_size sweep vs full ring averaging, bucket sizes, injected
per-hop latency -- on real NVLink (run under torch.distributed.run, one worker per GPU).

    python -m torch.distributed.run --nproc-per-node 4 tools/latency_sweep.py --out gpurun_out/sweep.json

For every group size m | n (m = n is Ring-SGD), every bucket size and every injected hop
delay, times one sesgd_sync_step through
  * the ring path (K5: the paper's Ring-AllReduce inside each group, 2(m-1) handshakes), and
  * the one-shot push path (K3: one handshake round), and
  * the two-shot push path (K4, the default: two handshake rounds),
as the max over ranks of the median CUDA-event time, and prints it next to the latency
model of Eq. 2 / Eq. 3 (sesgd_latency_model) evaluated with the measured per-hop latency
and push bandwidth.  Reproduces the SHAPE of the paper's Fig. 6 / "5x at 5 ms" argument
(P:7) on B200 NVLink; the paper's absolute numbers (K80, 1 Gbps) are context.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import SESGDEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-kib", default="64,1024,16384,131072,524288")
    ap.add_argument("--hops-us", default="0,100,5000")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tau-us", type=float, default=2.6, help="measured one-way hop (K7 ping-pong)")
    ap.add_argument("--nu-gbs", type=float, default=700.0, help="measured both-direction push GB/s")
    ap.add_argument("--out", default="gpurun_out/latency_sweep.json")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    n = world
    sizes = [int(s) * 1024 // 4 for s in a.sizes_kib.split(",")]  # fp32 elements
    hops = [int(h) * 1000 for h in a.hops_us.split(",")]
    rows = []
    stream = torch.cuda.current_stream()
    for m in [d for d in range(2, n + 1) if n % d == 0]:
        for path, pname in ((C.PATH_RING, "ring"), (C.PATH_ONESHOT, "oneshot"), (C.PATH_TWOSHOT, "twoshot")):
            for hop in hops:
                eng = SESGDEngine(n, m, sizes, rank=rank, world=world, path=path, hop_delay_ns=hop,
                                  timeout_ms=60000)
                for b, L in enumerate(sizes):
                    synth.fill_x0_device(eng.x(0, b).data_ptr(), L, 0, stream.cuda_stream)
                    synth.fill_grad_device(eng.g(0, b).data_ptr(), L, 0, rank, 0, stream.cuda_stream)
                t = 0
                for b, L in enumerate(sizes):
                    reps = a.reps if hop < 1_000_000 else 2
                    times = []
                    for _ in range(reps + 1):
                        eng.begin_iter(t)
                        t += 1
                        dist.barrier()
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        eng.sync_step(b, 0.1, 0.9, stream)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        times.append(e0.elapsed_time(e1) * 1e3)
                    us = statistics.median(times[1:])
                    tt = torch.tensor([us], device=dev, dtype=torch.float64)
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    model = C.sesgd_latency_model(n, m, 4.0 * L, a.nu_gbs * 1e9, a.tau_us * 1e-6 + hop * 1e-9)
                    rows.append({"n": n, "m": m, "path": pname, "bytes": 4 * L, "hop_us": hop / 1e3,
                                 "measured_us": float(tt.item()),
                                 "handshakes_per_call": (2 * (m - 1) if pname == "ring" else
                                                         {"oneshot": 1, "twoshot": 2}[pname] if m > 1 else 0),
                                 "model_group_us": model["sesgd_s"] * 1e6, "model_ring_n_us": model["ring_s"] * 1e6})
                eng.poll()
                eng.close()
                del eng
                torch.cuda.empty_cache()
                dist.barrier()
    if rank == 0:
        out = {"n": n, "tau_us_measured": a.tau_us, "nu_gbs_measured": a.nu_gbs, "rows": rows}
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)
        for r in rows:
            print(f"m={r['m']} {r['path']:7s} {r['bytes']/1024:9.0f} KiB hop {r['hop_us']:6.0f} us: "
                  f"{r['measured_us']:10.1f} us  (model {r['model_group_us']:10.1f} us, hs {r['handshakes_per_call']})")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""K7 probes on 2+ B200s (run under torch.distributed.run, one process per GPU).

Measures, through libsesgd's probe entry points (sesgd_probe_copy / sesgd_probe_pingpong):
  * local HBM copy bandwidth (read + write bytes / time),
  * NVLink pull (peer -> local) and push (local -> peer) bandwidth, one and both directions,
    over message sizes 64 KiB .. 1 GiB and CTA counts,
  * pull concurrent with a local HBM stream (can the exchange hide under the update?),
  * flag ping-pong round-trip latency (per-hop t_tau of Eq. 2).
Rank 0 prints one JSON object (and writes it to --out).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00433_b200 import sesgd as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/nvlink_probe.json")
    ap.add_argument("--gib", type=float, default=1.0)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    nbytes = int(a.gib * (1 << 30))
    buf = symm_mem.empty(2 * nbytes + 4096, dtype=torch.uint8, device=dev)
    buf.zero_()
    h = symm_mem.rendezvous(buf, dist.group.WORLD)
    dist.barrier()
    ptrs = list(h.buffer_ptrs)
    peer = (rank + 1) % world
    A = lambda r: ptrs[r]  # noqa: E731
    B = lambda r: ptrs[r] + nbytes  # noqa: E731
    FLAG = lambda r: ptrs[r] + 2 * nbytes  # noqa: E731
    s1 = torch.cuda.Stream(dev)
    s2 = torch.cuda.Stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    res = {"world": world, "sms": sms}

    def timed(fn, reps=5, stream=None):
        stream = stream or s1
        fn(stream)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(stream)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best * 1e-3

    def sync_all():
        torch.cuda.synchronize()
        dist.barrier()

    # 1. local copy
    t = timed(lambda s: C.sesgd_probe_copy(B(rank), A(rank), nbytes, sms * 4, s.cuda_stream))
    res["local_copy_gbs"] = 2 * nbytes / t / 1e9
    sync_all()
    # 2. pull / push, only rank 0 active
    out = {}
    for name, fn in [("pull", lambda s, c, n: C.sesgd_probe_copy(B(rank), A(peer), n, c, s.cuda_stream)),
                     ("push", lambda s, c, n: C.sesgd_probe_copy(B(peer), A(rank), n, c, s.cuda_stream))]:
        for ctas in (sms, 2 * sms, 4 * sms, 8 * sms):
            if rank == 0:
                t = timed(lambda s: fn(s, ctas, nbytes))
                out[f"{name}_1dir_ctas{ctas}_gbs"] = nbytes / t / 1e9
            sync_all()
        # both directions at once
        dist.barrier()
        t = timed(lambda s: fn(s, 4 * sms, nbytes))
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        out[f"{name}_bidir_per_dir_gbs"] = nbytes / float(tt.item()) / 1e9
        sync_all()
        # size sweep (1 direction)
        sweep = {}
        for sz in [1 << k for k in range(16, 31, 2)]:
            if sz > nbytes:
                break
            if rank == 0:
                t = timed(lambda s: fn(s, min(4 * sms, max(1, sz // (512 * 64))), sz), reps=20)
                sweep[str(sz)] = {"us": t * 1e6, "gbs": sz / t / 1e9}
            sync_all()
        out[f"{name}_size_sweep"] = sweep
    res.update(out)
    # 3b. push (both ranks at once, i.e. both directions) with few CTAs, alone and next to a
    #     local HBM stream on the remaining SMs: can the exchange hide under the update?
    half = nbytes // 2
    conc = {}
    for push_ctas in (8, 16, 32, 64, 148):
        dist.barrier()
        t_push = timed(lambda s: C.sesgd_probe_copy(B(peer), A(rank), half, push_ctas, s.cuda_stream))
        dist.barrier()
        t_loc = timed(lambda s: C.sesgd_probe_copy(B(rank) + half, A(rank) + half, half, 2 * sms,
                                                   s.cuda_stream))
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        C.sesgd_probe_copy(B(peer), A(rank), half, push_ctas, s1.cuda_stream)
        C.sesgd_probe_copy(B(rank) + half, A(rank) + half, half, 2 * sms, s2.cuda_stream)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize()
        conc[f"push_ctas{push_ctas}"] = {
            "push_alone_gbs": half / t_push / 1e9, "local_alone_gbs": 2 * half / t_loc / 1e9,
            "concurrent_push_us": e0.elapsed_time(e1) * 1e3, "concurrent_local_us": e0.elapsed_time(e2) * 1e3,
            "push_alone_us": t_push * 1e6, "local_alone_us": t_loc * 1e6}
        dist.barrier()
    res["push_bidir_with_local"] = conc
    # 3. pull concurrently with a local HBM stream
    if rank == 0:
        half = nbytes // 2
        t_pull = timed(lambda s: C.sesgd_probe_copy(B(rank), A(peer), half, 2 * sms, s.cuda_stream))
        t_loc = timed(lambda s: C.sesgd_probe_copy(B(rank) + half, A(rank) + half, half, 2 * sms, s.cuda_stream))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        C.sesgd_probe_copy(B(rank), A(peer), half, 2 * sms, s1.cuda_stream)
        C.sesgd_probe_copy(B(rank) + half, A(rank) + half, half, 2 * sms, s2.cuda_stream)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize()
        t_both = max(e0.elapsed_time(e1), e0.elapsed_time(e2)) * 1e-3
        res["overlap"] = {"pull_alone_us": t_pull * 1e6, "local_alone_us": t_loc * 1e6,
                          "concurrent_us": t_both * 1e6, "sum_us": (t_pull + t_loc) * 1e6}
    sync_all()
    # 4. ping-pong latency between rank 0 and rank 1
    if world >= 2 and rank < 2:
        out_ns = torch.zeros(1, dtype=torch.int64, device=dev)
        other = 1 - rank
        iters = 20000
        base = 1
        for rep in range(3):
            C.sesgd_probe_pingpong(FLAG(rank), FLAG(other), iters, rank == 0, base, out_ns.data_ptr(),
                                   s1.cuda_stream)
            base += 2 * iters + 2
            torch.cuda.synchronize()
        if rank == 0:
            ns = int(out_ns.item())
            res["pingpong"] = {"iters": iters, "rtt_ns": ns / iters, "one_way_hop_ns": ns / iters / 2}
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        print(json.dumps(res, indent=1))
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

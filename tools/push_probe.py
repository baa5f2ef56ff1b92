#!/usr/bin/env python
"""Both-direction NVLink push bandwidth vs CTA count and threads per CTA (K7 probe).

    python -m torch.distributed.run --nproc-per-node 2 tools/push_probe.py

Every rank pushes `--mib` MiB from its own buffer into the peer's buffer at the same time
(sesgd_probe_copy, 128-bit stores), for CTA counts x threads per CTA; prints GB/s per
direction and per CTA.  Also the same with an L2-resident (16 MiB, re-read) source.
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
    ap.add_argument("--mib", type=int, default=512)
    ap.add_argument("--out", default="gpurun_out/push_probe.json")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    nbytes = a.mib << 20
    buf = symm_mem.empty(2 * nbytes, dtype=torch.uint8, device=dev)
    buf.zero_()
    h = symm_mem.rendezvous(buf, dist.group.WORLD)
    dist.barrier()
    ptrs = list(h.buffer_ptrs)
    peer = (rank + 1) % world
    src, dst = ptrs[rank], ptrs[peer] + nbytes
    s = torch.cuda.Stream(dev)
    res = {}
    for threads in (128, 256, 512):
        for ctas in (8, 16, 32, 48, 64, 96):
            code = ctas | ((threads // 32) << 16)
            for name, sz in (("hbm_src", nbytes), ("l2_src", 16 << 20)):
                reps = 1 if name == "hbm_src" else nbytes // sz
                dist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                C.sesgd_probe_copy(dst, src, sz, code, s.cuda_stream)  # warm
                torch.cuda.synchronize()
                dist.barrier()
                e0.record(s)
                for _ in range(reps):
                    C.sesgd_probe_copy(dst, src, sz, code, s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) * 1e-3
                tt = torch.tensor([t], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                gbs = sz * reps / float(tt.item()) / 1e9
                res[f"{name}_t{threads}_c{ctas}"] = {"gbs_per_dir": gbs, "gbs_per_cta": gbs / ctas}
    if rank == 0:
        print(json.dumps(res, indent=1))
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

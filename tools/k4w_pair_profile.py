#!/usr/bin/env python
"""ncu harness for the multi-GPU exchange kernels K4W / K4W-M: two loopback virtual ranks (the
ResNet-50 cfg-2 buckets; n = m = 2, one worker each = K4W, or n = 8, m = 2, four workers each =
K4W-M, the cfg-2 shape at N = 2) on ONE GPU, each iteration as ONE launch of both ranks' grids
(sesgd_sync_all_pair), so ncu -- which serialises launches and replays them -- can capture the
whole exchange:

    ncu --set full -k regex:k4w_pair -s 3 -c 1 python tools/k4w_pair_profile.py [iters] [n]
    ncu --set full -k regex:k4w_multi_pair -s 3 -c 1 python tools/k4w_pair_profile.py 10 8

Without ncu it prints the mean CUDA-event time of a pair launch.  The peers' pushes land in local
memory here (no NVLink), so the DRAM counters include the exchange traffic that NVLink carries
on two GPUs; DESIGN.md 5 states the per-launch algorithmic bytes to compare with."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import LoopbackGroup  # noqa: E402
from paper_2007_00433_b200.workloads import WORKLOADS  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    split = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    buckets = list(WORKLOADS["resnet50"])
    opts = {C.OPT_PROTOCOL: 2} | ({C.OPT_WS_SPLIT: split} if split else {})
    grp = LoopbackGroup(2, n, 2, buckets, seed=42, options=opts)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for e in grp:
        for s, w in enumerate(e.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_x0_device(e.x(s, b).data_ptr(), L, int(offs[b]), e.stream.cuda_stream)
                synth.fill_grad_device(e.g(s, b).data_ptr(), L, int(offs[b]), w, 0, e.stream.cuda_stream)
    grp.synchronize()
    for t in range(3):
        grp.step_pair(t, 0.1, 0.9)
    grp.synchronize()
    s0 = grp[0].stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    for t in range(3, 3 + iters):
        grp.step_pair(t, 0.1, 0.9)
    e1.record(s0)
    grp.synchronize()
    grp.poll()
    L = sum(buckets)
    ms = e0.elapsed_time(e1) / iters
    print(json.dumps({"n": n, "workers_per_rank": n // 2, "ms_per_pair_launch": ms,
                      "algo_hbm_bytes_per_launch": n * 20 * L, "launches": iters}))
    grp.close()


if __name__ == "__main__":
    main()

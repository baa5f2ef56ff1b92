#!/usr/bin/env python
"""Two ranks on two GPUs WITHOUT NCCL: rank 0 is this process, rank 1 a spawned child; the
workspaces are shared through CUDA IPC (torch.multiprocessing) and attached with
sesgd_attach_peers.  Made for ncu: `ncu --target-processes application-only ... python
tools/ipc_pair.py ...` profiles rank 0's kernels while rank 1 runs unprofiled and concurrently
(a metric set that fits one pass needs no kernel replay, so the peer handshakes are the normal
ones).  Without ncu it prints rank 0's mean kernel time (CUDA events).

    python tools/ipc_pair.py --workers 2 --gsize 2 --protocol 2 --iters 20
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(rank, a, q_out, q_in, bar):
    import synth
    from paper_2007_00433_b200 import sesgd as C
    from paper_2007_00433_b200.engine import SESGDEngine
    from paper_2007_00433_b200.workloads import WORKLOADS
    torch.cuda.set_device(rank)
    buckets = list(WORKLOADS[a.workload])
    opts = {C.OPT_PROTOCOL: a.protocol} if a.protocol else {}
    eng = SESGDEngine(a.workers, a.gsize, buckets, seed=42, rank=rank, world=2, path=a.path,
                      manual_peers=True, options=opts)
    q_out.put(eng.workspace)           # shared with the peer through CUDA IPC
    peer = q_in.get()
    ptrs = [eng.workspace.data_ptr(), peer.data_ptr()] if rank == 0 else [peer.data_ptr(), eng.workspace.data_ptr()]
    eng.attach_peers(ptrs)
    st = torch.cuda.current_stream()
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for s, w in enumerate(eng.local_workers):
        for b, L in enumerate(buckets):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, int(offs[b]), st.cuda_stream)
            synth.fill_grad_device(eng.g(s, b).data_ptr(), L, int(offs[b]), w, 0, st.cuda_stream)
    torch.cuda.synchronize()
    bar.wait()
    for t in range(a.warmup):
        eng.step(t, 0.1, 0.9)
    torch.cuda.synchronize()
    bar.wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.warmup, a.warmup + a.iters):
        eng.step(t, 0.1, 0.9)
    e1.record()
    torch.cuda.synchronize()
    eng.poll()
    bar.wait()
    ms = e0.elapsed_time(e1) / a.iters
    del peer
    bar.wait()
    eng.close()
    return ms


def child(a, q_out, q_in, bar):
    run(1, a, q_out, q_in, bar)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workers", type=int, default=2)
    p.add_argument("--gsize", type=int, default=2)
    p.add_argument("--protocol", type=int, default=0)
    p.add_argument("--path", type=int, default=4)
    p.add_argument("--workload", default="resnet50")
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    a = p.parse_args()
    ctx = mp.get_context("spawn")
    q01, q10 = ctx.Queue(), ctx.Queue()
    bar = ctx.Barrier(2)
    proc = ctx.Process(target=child, args=(a, q10, q01, bar))
    proc.start()
    ms = run(0, a, q01, q10, bar)
    proc.join()
    print(json.dumps({"ms_per_step_rank0": ms, "workers": a.workers, "gsize": a.gsize,
                      "protocol": a.protocol, "workload": a.workload}))
    return proc.exitcode


if __name__ == "__main__":
    sys.exit(main())

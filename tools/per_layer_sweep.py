#!/usr/bin/env python
"""BASELINE config 4, per-layer half: ResNet-50 synchronised tensor by tensor (161 buckets, one
sesgd_sync_step each -- the paper's per-layer handshakes, "50*2*(16-1) = 1500 handshakes",
P:108-112, Table 1), SESGD (group_size m < n) against Ring-SGD (m = n), at injected per-hop
latencies, one worker per GPU (torch.distributed.run), or R virtual ranks on one GPU (--loopback R).

    python -m torch.distributed.run --nproc-per-node 4 tools/per_layer_sweep.py --out gpurun_out/pl.json
    python tools/per_layer_sweep.py --loopback 4 --out gpurun_out/pl_loop.json

Per (m, path, hop): W warm-up iterations, then K timed iterations three ways -- eager (161
launches per iteration from Python), as ONE captured CUDA graph of the same K iterations (the
kernels and their arguments are identical; the graph removes the host launch overhead; single
use), and with the device-resident iteration state (SESGD_OPT_DEVICE_ITER): ONE iteration
captured once and the graph replayed K times, t / groups / call history advancing on the device
-- max over ranks.  The per-hop latency tau is measured in the same run (sesgd_measure_hop, K7 ping-pong
through the workspaces), and every row carries the Eq. 2 / Eq. 3 prediction
(sesgd_latency_model per tensor, summed over the 161 tensors) and the device-counted flag
stores per iteration.  Paths: ring = K5, the paper's Ring-AllReduce inside each group (2(m-1)
handshakes per tensor); twoshot = K4 (two handshake rounds per tensor, value-carried).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import LoopbackGroup, SESGDEngine  # noqa: E402
from paper_2007_00433_b200.workloads import WORKLOADS  # noqa: E402


class Ranks:
    """the R engines this process drives: one (torch.distributed) or R virtual ranks (loopback)"""

    def __init__(self, a, n, m, buckets, path, hop_ns):
        self.loop = a.loopback > 0
        kw = dict(seed=42, path=path, hop_delay_ns=hop_ns, timeout_ms=120000)
        if self.loop:
            self.grp = LoopbackGroup(a.loopback, n, m, buckets, **kw)
            self.engs = list(self.grp)
        else:
            self.grp = None
            self.engs = [SESGDEngine(n, m, buckets, rank=a.rank, world=a.world, **kw)]
        offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
        for e in self.engs:
            st = e.default_stream().cuda_stream
            for s, w in enumerate(e.local_workers):
                for b, L in enumerate(buckets):
                    synth.fill_x0_device(e.x(s, b).data_ptr(), L, int(offs[b]), st)
                    synth.fill_grad_device(e.g(s, b).data_ptr(), L, int(offs[b]), w, 0, st)
        self.sync()

    def sync(self):
        torch.cuda.synchronize()
        if not self.loop and torch.distributed.is_initialized():
            torch.distributed.barrier()
            torch.cuda.synchronize()

    def iteration(self, t, nb):
        for e in self.engs:
            e.begin_iter(t)
            for b in range(nb):
                e.sync_step(b, 0.1, 0.9)

    def close(self):
        for e in self.engs:
            e.poll()
            e.close()


def max_over_ranks(v):
    if torch.distributed.is_initialized():
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    return v


def measure_tau(a, n):
    """one-way flag hop between rank 0 and rank 1 through the workspaces (sesgd_measure_hop)"""
    r = Ranks(a, n, n, [4096], C.PATH_TWOSHOT, 0)
    if r.loop:
        e0, e1 = r.engs[0], r.engs[1]
        e0.measure_hop(1, 5000, True)
        e1.measure_hop(0, 5000, False)
    elif a.rank < 2:
        r.engs[0].measure_hop(1 - a.rank, 5000, a.rank == 0)
    r.sync()
    hop = max_over_ranks(r.engs[0].stats(0)["hop_ns"] if (r.loop or a.rank == 0) else 0.0)
    r.close()
    return hop * 1e-9


def time_config(a, n, m, path, hop_ns, buckets, K, W):
    nb = len(buckets)
    r = Ranks(a, n, m, buckets, path, hop_ns)
    t = 0
    for _ in range(W):
        r.iteration(t, nb)
        t += 1
    r.sync()
    st0 = r.engs[0].stats(0)
    # eager
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = r.engs[0].default_stream()
    ev0.record(s0)
    for _ in range(K):
        r.iteration(t, nb)
        t += 1
    for e in r.engs[1:]:  # loopback: rank 0's end event after every virtual rank's work
        s0.wait_stream(e.default_stream())
    ev1.record(s0)
    r.sync()
    eager_ms = max_over_ranks(ev0.elapsed_time(ev1)) / K
    st1 = r.engs[0].stats(0)
    # the same K iterations captured into one CUDA graph (per virtual rank: its own stream)
    graphs = []
    for e in r.engs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=e.stream if r.loop else None):  # (not the legacy stream)
            for k in range(K):
                e.begin_iter(t + k)
                for b in range(nb):
                    e.sync_step(b, 0.1, 0.9, torch.cuda.current_stream())
        graphs.append(g)
    t += K
    r.sync()
    ev0.record(s0)
    for e, g in zip(r.engs, graphs):
        with torch.cuda.stream(e.default_stream()):
            g.replay()
    for e in r.engs[1:]:
        s0.wait_stream(e.default_stream())
    ev1.record(s0)
    r.sync()
    graph_ms = max_over_ranks(ev0.elapsed_time(ev1)) / K
    # device-resident iteration state (SESGD_OPT_DEVICE_ITER): ONE iteration captured once, the
    # graph replayed K times -- t, the groups and the call history advance on the device
    for e in r.engs:
        e.set_device_iter(True)
    dgraphs = [e.capture_iteration(0.1, 0.9, None, fused=False) for e in r.engs]
    for e, g in zip(r.engs, dgraphs):  # one warm-up replay
        e.replay_iteration(g)
    r.sync()
    ev0.record(s0)
    for _ in range(K):
        for e, g in zip(r.engs, dgraphs):
            e.replay_iteration(g)
    for e in r.engs[1:]:
        s0.wait_stream(e.default_stream())
    ev1.record(s0)
    r.sync()
    devgraph_ms = max_over_ranks(ev0.elapsed_time(ev1)) / K
    for e in r.engs:
        e.set_device_iter(False)
    flags_per_iter = (st1["dev_flag_stores"] - st0["dev_flag_stores"]) / K
    rounds = st1["handshake_rounds"]
    r.close()
    return {"eager_ms_per_iter": eager_ms, "graph_ms_per_iter": graph_ms,
            "device_iter_graph_ms_per_iter": devgraph_ms,
            "launches_per_iter": nb, "handshake_rounds_per_tensor": rounds,
            "device_flag_stores_per_iter_rank0": flags_per_iter}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--loopback", type=int, default=0, help="R virtual ranks on one GPU (no torchrun)")
    ap.add_argument("--hops-us", default="0,100")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--nu-gbs", type=float, default=770.0)
    ap.add_argument("--out", default="gpurun_out/per_layer_sweep.json")
    a = ap.parse_args()
    if a.loopback:
        a.rank, a.world = 0, a.loopback
        torch.cuda.set_device(0)
        n = a.loopback
    else:
        a.rank, a.world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", a.rank)))
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        n = a.world
    buckets = list(WORKLOADS["resnet50_per_layer"])
    tau = measure_tau(a, n)
    rows = []
    for hop_us in [float(h) for h in a.hops_us.split(",")]:
        hop_ns = int(hop_us * 1000)
        K = a.iters if hop_us < 1000 else 1
        for m in [d for d in range(2, n + 1) if n % d == 0]:
            for path, pname in ((C.PATH_RING, "ring"), (C.PATH_TWOSHOT, "twoshot")):
                res = time_config(a, n, m, path, hop_ns, buckets, K, min(a.warmup, K))
                model = {"ring_s": 0.0, "sesgd_s": 0.0}
                for L in buckets:  # Eq. 2 / Eq. 3 per tensor with tau = measured hop + injected hop
                    c = C.sesgd_latency_model(n, m, 4.0 * L, a.nu_gbs * 1e9, tau + hop_ns * 1e-9)
                    model["ring_s"] += c["ring_s"]
                    model["sesgd_s"] += c["sesgd_s"]
                row = {"n": n, "m": m, "path": pname, "hop_us": hop_us, "iters": K,
                       "handshakes_per_tensor_eq3": 2 * (m - 1), "handshakes_per_tensor_ring_n": 2 * (n - 1),
                       "model_ms_per_iter_eq3": model["sesgd_s"] * 1e3,
                       "model_ms_per_iter_ring_over_n": model["ring_s"] * 1e3, **res}
                rows.append(row)
                if a.rank == 0:
                    print(json.dumps(row), flush=True)
    out = {"what": "per-layer ResNet-50 (161 tensors), one sync per tensor; eager vs one captured CUDA graph",
           "tau_measured_s": tau, "transport": f"loopback x{a.loopback}" if a.loopback else f"NVLink x{n}",
           "rows": rows}
    if a.rank == 0:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

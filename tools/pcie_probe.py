#!/usr/bin/env python
"""PCIe bound of bench.py's e2e leg: pinned host <-> HBM copy time for the bytes one step moves.

The e2e step (sesgd_sync_all_host) copies every worker's gradient in (H2D) and updated parameters
out (D2H): 8 workers x 25,557,032 fp32 each way at cfg 2, N = 1.  This probe times, with CUDA
events, the same bytes as H2D alone, D2H alone and both directions at once on two streams (what
the library's pipelined call overlaps), so the e2e number can be read against its own roofline.

    python tools/pcie_probe.py [--mb 817.8] [--reps 5] > gpurun_out/pcie_probe.json
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=8 * 25557032 * 4 / 1e6)
    ap.add_argument("--pieces", type=int, default=40)  # 8 workers x 5 buckets
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = int(a.mb * 1e6 / 4) // a.pieces * a.pieces
    dev = torch.device("cuda:0")
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float32, device=dev)
    d_out = torch.ones(n, dtype=torch.float32, device=dev)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    step = n // a.pieces

    def h2d():
        with torch.cuda.stream(s_in):
            for p in range(a.pieces):
                d_in[p * step:(p + 1) * step].copy_(h_in[p * step:(p + 1) * step], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s_out):
            for p in range(a.pieces):
                h_out[p * step:(p + 1) * step].copy_(d_out[p * step:(p + 1) * step], non_blocking=True)

    def timed(fn):
        best = []
        for _ in range(a.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            s_in.wait_stream(cur)
            s_out.wait_stream(cur)
            fn()
            cur.wait_stream(s_in)
            cur.wait_stream(s_out)
            e1.record(cur)
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1))
        return sorted(best[1:])[len(best[1:]) // 2]  # median after one warm-up

    t_in, t_out = timed(h2d), timed(d2h)
    t_both = timed(lambda: (h2d(), d2h()))
    nbytes = n * 4
    print(json.dumps({
        "bytes_each_way": nbytes, "pieces": a.pieces,
        "h2d_ms": t_in, "h2d_gbs": nbytes / t_in / 1e6,
        "d2h_ms": t_out, "d2h_gbs": nbytes / t_out / 1e6,
        "both_ms": t_both, "both_gbs_per_dir": nbytes / t_both / 1e6,
        "device": torch.cuda.get_device_name(0),
    }))


if __name__ == "__main__":
    main()

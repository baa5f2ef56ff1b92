"""Per-rank body of the SESGDDataParallel test (launched by tests/test_gpu_ddp.py via
torch.distributed.run, one worker per GPU).

Trains a small MLP for T steps through SESGDDataParallel (parameters and gradients are views
into the engine's fusion buffers; every bucket's SESGD step is enqueued from a gradient hook on
a side stream during backward).  After every step rank 0 gathers each worker's x, v before the
step and the gradients autograd accumulated, replays the step with the CPU oracle (oracle.step,
binary32 op order) and checks the gathered x, v after the step bit for bit."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402  (test infrastructure: the replay checker)
from paper_2007_00433_b200.ddp import SESGDDataParallel  # noqa: E402

LR, MU = 0.05, 0.9


def gather(t):
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.stack([o.cpu().numpy() for o in out])


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gsize", type=int, required=True)
    p.add_argument("--iters", type=int, default=4)
    p.add_argument("--overlap", type=int, default=1)
    p.add_argument("--mode", type=int, default=0)
    p.add_argument("--static", type=int, default=0)
    p.add_argument("--graph", type=int, default=0)  # steps >= 2 replay one captured step (enable_graphs)
    p.add_argument("--out", required=True)
    a = p.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)

    torch.manual_seed(rank)  # distinct random init per rank: SESGDDataParallel broadcasts rank 0's x_0
    model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 512),
                                torch.nn.ReLU(), torch.nn.Linear(512, 10)).to(dev)
    # small caps so the MLP spans three buckets (the last layer first, as DDP orders them)
    ddp = SESGDDataParallel(model, world, a.gsize, lr=LR, momentum=MU, rank=rank, world=world,
                            mode=a.mode, first_bucket_bytes=16 << 10, bucket_bytes=256 << 10,
                            overlap=bool(a.overlap), static_graph=bool(a.static))
    eng = ddp.engine
    nb = len(ddp.bucket_params)
    X_init = gather(eng.x_flat[0])  # identical x_0 on every worker (Alg.1 line 1)
    assert np.array_equal(X_init, np.broadcast_to(X_init[:1], X_init.shape)), "x_0 differs across ranks"
    log = []
    inp = torch.zeros(64, 256, device=dev)
    lab = torch.zeros(64, dtype=torch.long, device=dev)
    graph = None
    for t in range(a.iters):
        torch.cuda.synchronize()
        x_prev, v_prev = eng.x_flat[0].clone(), eng.v_flat[0].clone()
        gen = torch.Generator(device=dev).manual_seed(1000 * t + rank)
        inp.copy_(torch.randn(64, 256, device=dev, generator=gen))
        lab.copy_(torch.randint(0, 10, (64,), device=dev, generator=gen))
        if a.graph and t == 2:  # after two eager steps: capture the whole step once (enable_graphs)
            # drop the last eager loss: its autograd graph keeps AccumulateGrad nodes bound to the
            # legacy stream, which the captured backward would then have to join (illegal in capture)
            loss = None
            ddp.enable_graphs()
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(graph, stream=cap):
                ddp.begin_step()
                static_loss = F.cross_entropy(model(inp), lab)
                static_loss.backward()
                ddp.finish_step()
            torch.cuda.current_stream().wait_stream(cap)
        if graph is not None:
            graph.replay()
            loss = static_loss
            in_bwd = len(ddp.bucket_params)
        else:
            ddp.begin_step(t)
            loss = F.cross_entropy(model(inp), lab)
            loss.backward()
            in_bwd = ddp.launched_in_backward
            ddp.finish_step()
        torch.cuda.synchronize()
        eng.poll()
        X0, V0, G = gather(x_prev), gather(v_prev), gather(eng.g_flat[0])
        X1, V1 = gather(eng.x_flat[0]), gather(eng.v_flat[0])
        if rank == 0:
            _, canon, _ = oracle.groups(42, t, world, a.gsize)
            x, v = X0.copy(), V0.copy()
            oracle.step(world, a.gsize, canon, x, v, G, LR, MU, a.mode)
            bad_x = int(np.count_nonzero(x.view(np.uint32) != X1.view(np.uint32)))
            bad_v = int(np.count_nonzero(v.view(np.uint32) != V1.view(np.uint32)))
            log.append((t, float(loss), bad_x, bad_v, in_bwd, float(np.abs(G).max()), len(ddp._hooks)))
    if graph is not None:  # release the captured graph before the engine and the process group go
        torch.cuda.synchronize()
        del graph, static_loss
    # model parameters are the engine's x: the module sees the synchronised values
    first = next(model.parameters())
    assert first.data_ptr() >= eng.x_flat[0].data_ptr()
    if rank == 0:
        np.save(a.out, np.array(log, dtype=np.float64))
        print("buckets", nb, "log", log)
    dist.barrier()
    ddp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

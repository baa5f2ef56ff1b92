"""BASELINE config 5 / SURVEY NEXT-1: ResNet-50 synthetic-data training, random init, one worker
per GPU, SESGD (group_size m) with backward/sync overlap vs the NCCL Ring-SGD baseline (torch
DistributedDataParallel, all-reduce + torch SGD momentum).

Arms, each timed with CUDA events on the compute stream between a barrier + synchronize, max
over ranks:
  compute   forward + backward only (no synchronisation, no update): the floor
  sesgd     SESGDDataParallel, every bucket's sesgd_sync_step enqueued from a gradient hook on a
            side stream during backward (the fused average + momentum update is the optimizer)
  sesgd_seq the same engine, all buckets synced after backward (no overlap)
  ddp       torch DDP (NCCL ring all-reduce, 25 MiB buckets, gradient_as_bucket_view) +
            torch.optim.SGD(momentum, foreach): Ring-SGD, the paper's baseline
  compute_accum  the floor with gradients accumulated in place into one flat buffer (what every
            bucketed data-parallel wrapper, torch DDP's gradient_as_bucket_view included, pays)
  compute_hooks  the floor plus a no-op Python hook per parameter
  sesgd_graph   sesgd, but after the eager warm-up the whole step (zero grads, device-side
            begin_iter, forward, backward with the hook-launched bucket syncs on the side stream,
            finish) is captured once with torch.cuda.graph (SESGD_OPT_DEVICE_ITER) and replayed
The sync hidden fraction is (sesgd_seq - sesgd) / (sesgd_seq - floor), floor = compute_accum when
timed, else compute.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/train_bench.py
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.ddp import SESGDDataParallel  # noqa: E402

LR, MU = 0.1, 0.9


def build_model(dev, channels_last):
    import torchvision
    torch.manual_seed(0)  # identical random init on every worker
    model = torchvision.models.resnet50().to(dev)
    if channels_last:
        model = model.to(memory_format=torch.channels_last)
    return model


def time_arm(arm, a, rank, world, dev, images, labels):
    model = build_model(dev, a.channels_last)
    model.train()
    ddp = opt = None
    net = model
    if arm in ("sesgd", "sesgd_seq", "sesgd_graph"):
        ddp = SESGDDataParallel(model, world, min(a.gsize, world), lr=LR, momentum=MU, rank=rank,
                                world=world, overlap=(arm != "sesgd_seq"), static_graph=bool(a.static),
                                engine_options={} if not a.grid else {C.OPT_GRID: a.grid})
    elif arm == "compute_hooks":  # the floor plus one no-op Python hook per parameter
        hooks = [p.register_post_accumulate_grad_hook(lambda p: None) for p in model.parameters()]
    elif arm == "compute_accum":  # the floor with gradients accumulated in place into a flat buffer
        params = list(model.parameters())
        flat = torch.zeros(sum(p.numel() for p in params), device=dev)
        off = 0
        for p in params:
            p.grad = flat[off:off + p.numel()].view(p.size()) if p.is_contiguous() else \
                flat[off:off + p.numel()].as_strided(p.size(), p.stride())
            off += p.numel()
    elif arm == "ddp":
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[dev.index],
                                                        gradient_as_bucket_view=True)
        opt = torch.optim.SGD(model.parameters(), lr=LR, momentum=MU, foreach=True)
    amp = torch.autocast("cuda", dtype=torch.bfloat16, enabled=a.amp == "bf16")

    def step(t):
        if ddp is not None:
            ddp.begin_step(t)
        elif opt is not None:
            opt.zero_grad(set_to_none=False)
        elif arm == "compute_accum":
            flat.zero_()
        else:
            for p in model.parameters():
                p.grad = None
        with amp:
            loss = F.cross_entropy(net(images), labels)
        loss.backward()
        if ddp is not None:
            ddp.finish_step()
        elif opt is not None:
            opt.step()
        return loss

    for t in range(a.warmup):
        step(t)
    if arm == "sesgd_graph":  # capture one step, replay it every step
        torch.cuda.synchronize()
        ddp.enable_graphs()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(torch.cuda.current_stream())
        cap_amp = torch.autocast("cuda", dtype=torch.bfloat16, enabled=a.amp == "bf16", cache_enabled=False)
        with torch.cuda.graph(graph, stream=cap):
            ddp.begin_step()
            with cap_amp:
                static_loss = F.cross_entropy(net(images), labels)
            static_loss.backward()
            ddp.finish_step()
        torch.cuda.current_stream().wait_stream(cap)

        def step(t):  # noqa: F811 -- the replayed step
            graph.replay()
            return static_loss

        for t in range(2):
            step(t)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for t in range(a.warmup, a.warmup + a.steps):
        loss = step(t)
    e1.record()
    host = time.perf_counter() - w0  # enqueue time (the GPU may still be running)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    out = {"ms_per_step": float(ms), "images_per_s": a.batch * world * 1000.0 / float(ms),
           "loss": float(loss.detach()), "wall_ms_per_step": 1000.0 * wall / a.steps,
           "host_enqueue_ms_per_step": 1000.0 * host / a.steps}
    if arm == "compute_hooks":
        for h in hooks:
            h.remove()
    if ddp is not None:
        ddp.engine.poll()
        out["buckets"] = len(ddp.bucket_params)
        out["launched_in_backward"] = ddp.launched_in_backward
        ddp.close()
    del net, model, opt
    torch.cuda.empty_cache()
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--arms", default="compute,sesgd,sesgd_seq,ddp")
    p.add_argument("--batch", type=int, default=64, help="images per GPU")
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--gsize", type=int, default=2)
    p.add_argument("--amp", default="bf16", choices=["bf16", "none"])
    p.add_argument("--channels-last", type=int, default=1)
    p.add_argument("--grid", type=int, default=0, help="SESGD CTAs per launch (0 = library default)")
    p.add_argument("--static", type=int, default=1, help="SESGDDataParallel static_graph")
    p.add_argument("--out", default="")
    a = p.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    torch.backends.cudnn.benchmark = True
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    images = torch.randn(a.batch, 3, 224, 224, device=dev, generator=gen)
    if a.channels_last:
        images = images.contiguous(memory_format=torch.channels_last)
    labels = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
    res = {}
    for arm in a.arms.split(","):
        res[arm] = time_arm(arm, a, rank, world, dev, images, labels)
    if rank == 0:
        line = {"workload": "resnet50 synthetic training", "n_gpus": world, "group_size": a.gsize,
                "batch_per_gpu": a.batch, "amp": a.amp, "grid": a.grid, "static_graph": a.static,
                "channels_last": a.channels_last, "steps": a.steps,
                "warmup": a.warmup, "arms": res}
        floor = "compute_accum" if "compute_accum" in res else "compute"
        if all(k in res for k in (floor, "sesgd", "sesgd_seq")):
            line["floor_arm"] = floor
            sync = res["sesgd_seq"]["ms_per_step"] - res[floor]["ms_per_step"]
            hid = res["sesgd_seq"]["ms_per_step"] - res["sesgd"]["ms_per_step"]
            line["sync_exposed_ms_no_overlap"] = sync
            line["sync_hidden_fraction"] = hid / sync if sync > 0 else None
        if "ddp" in res and "sesgd" in res:
            line["sesgd_over_ddp_images_per_s"] = res["sesgd"]["images_per_s"] / res["ddp"]["images_per_s"]
        print(json.dumps(line))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(line, f, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

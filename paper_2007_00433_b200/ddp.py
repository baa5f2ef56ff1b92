"""SESGDDataParallel: the gradient fusion buffer + backward/sync overlap (SURVEY NEXT-1,
BASELINE config 5), the paper's integration "imitating the PyTorch DistributedDataParallel
module and using register_hook ... to implement the overlap between computation and
communication" (Fig. 1b).

One SESGD worker per process / GPU.  The module's parameters and gradients become views into
the SESGDEngine's flat per-bucket fp32 buffers (no pack copy): buckets in reverse registration
order, the first capped at 1 MiB and the rest at 25 MiB, as torch DDP does.  A
post-accumulate-grad hook per parameter counts the parameters of each bucket; once a bucket's
gradients are complete (and every earlier bucket's, so every rank issues the same bucket
order), `sesgd_sync_step(bucket)` is enqueued on a side stream behind an event of the backward
stream, overlapping the rest of backward.  The SESGD kernel IS the optimizer step: it applies
momentum SGD and the group average to the parameters in place (Eq. 6), so no torch optimizer
runs.  `finish_step()` makes the compute stream wait for the side stream.  With
static_graph=True (torch DDP's option of the same name) the first step records the gradient
order and later steps keep one hook per bucket, on its last-accumulated parameter.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import sesgd as C
from .engine import SESGDEngine
from .workloads import assign_buckets


class BucketReadiness:
    """Host logic of the overlap: a countdown of the gradients each bucket still waits for; a
    bucket is released only when it and every earlier bucket are complete, so every rank
    enqueues the same bucket sequence (peers' kernels wait on the same bucket)."""

    def __init__(self, counts):
        self.counts = [int(c) for c in counts]
        self.reset()

    def reset(self, counts=None) -> None:
        if counts is not None:
            self.counts = [int(c) for c in counts]
        self.pending = list(self.counts)
        self.next = 0

    def arrive(self, b: int):
        """One gradient of bucket b accumulated; returns the buckets now released, in order."""
        if self.pending[b] <= 0:
            raise RuntimeError(f"bucket {b} received more gradients than it holds")
        self.pending[b] -= 1
        return self.release()

    def release(self):
        out = []
        while self.next < len(self.pending) and self.pending[self.next] == 0:
            out.append(self.next)
            self.next += 1
        return out

    def force_all(self):
        """No hooks (overlap off): every remaining bucket, in order."""
        self.pending = [0] * len(self.pending)
        return self.release()

    def done(self) -> bool:
        return self.next == len(self.pending)


def _like(flat: torch.Tensor, p: torch.Tensor) -> torch.Tensor:
    """A view of the flat slice with p's shape and, when p is dense in channels_last, its
    strides (so cuDNN sees the weight layout it was given)."""
    if p.dim() == 4 and not p.is_contiguous() and p.is_contiguous(memory_format=torch.channels_last):
        return flat.as_strided(p.size(), p.stride())
    return flat.view(p.size())


class SESGDDataParallel:
    def __init__(self, module: torch.nn.Module, n: int, group_size: int, *, lr: float, momentum: float,
                 rank: int = 0, world: int = 1, seed: int = 42, mode: int = C.MODE_PARAM_AVG,
                 first_bucket_bytes: int = 1 << 20, bucket_bytes: int = 25 << 20, process_group=None,
                 overlap: bool = True, static_graph: bool = False,
                 engine_options: Optional[dict] = None, engine: Optional[SESGDEngine] = None):
        """engine: an SESGDEngine to run on instead of creating one -- e.g. a loopback virtual
        rank of engine.LoopbackGroup (one worker each, bucket sizes as this module's buckets), so
        several replicas in ONE process on ONE GPU train through the NVLink-path kernels; the
        caller then gives every replica the same x_0 (there is no process group to broadcast over)"""
        if n != world:
            raise ValueError("SESGDDataParallel runs one worker per process (n == world size)")
        if overlap and (engine_options or {}).get(C.OPT_P2P_VARIANT, 0) >= 1:
            # the SM-specialised one-shot kernel (K3 split) has COMM and COMPUTE CTAs of the same
            # grid wait on each other: launched on a side stream while backward kernels hold SMs,
            # part of the grid may not become resident (sesgd_capi.cu launches it cooperatively,
            # so it fails instead of hanging) -- the overlap uses the default K4 path
            raise ValueError("overlap=True needs the default P2P layout (SESGD_OPT_P2P_VARIANT 0)")
        self.module = module
        self.lr, self.momentum = lr, momentum
        self.overlap = overlap
        self.params = [p for p in module.parameters() if p.requires_grad]
        sizes = [p.numel() for p in self.params]
        self.bucket_params = assign_buckets(sizes, first_bucket_bytes, bucket_bytes)
        bucket_sizes = [sum(sizes[i] for i in b) for b in self.bucket_params]
        dev = self.params[0].device
        if engine is not None:
            if engine.r != 1 or engine.bucket_sizes != bucket_sizes or engine.n != n or engine.m != group_size:
                raise ValueError("the given engine must hold one worker with this module's buckets")
            self.engine = engine
        else:
            self.engine = SESGDEngine(n, group_size, bucket_sizes, seed=seed, mode=mode, rank=rank,
                                      world=world, device=dev.index, process_group=process_group,
                                      options=engine_options)
        self._own_engine = engine is None
        self.bucket_of = {}
        with torch.no_grad():
            for b, idxs in enumerate(self.bucket_params):
                off = 0
                xb, gb = self.engine.x(0, b), self.engine.g(0, b)
                for i in idxs:
                    p = self.params[i]
                    k = p.numel()
                    view, gview = _like(xb[off:off + k], p), _like(gb[off:off + k], p)
                    view.copy_(p.data)
                    p.data = view   # parameter lives in the fusion buffer
                    p.grad = gview  # gradient accumulates into it (in place)
                    self.bucket_of[id(p)] = b
                    off += k
        if world > 1 and self._own_engine:
            self._broadcast_state(module)
        self.ready = BucketReadiness([len(b) for b in self.bucket_params])
        self.launched_in_backward = 0
        self.side = torch.cuda.Stream(dev)
        self.done_event = torch.cuda.Event()
        self.t = 0
        # static_graph (as torch DDP's): the autograd graph and its gradient order are the same
        # every step, so after the first step only the last-accumulated parameter of each bucket
        # keeps a hook (one Python call per bucket instead of one per parameter)
        self.static_graph = static_graph
        self._order: list = []
        self._hooks = {}
        if overlap:
            self._hooks = {id(p): p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params}
        self._hooked = [len(b) for b in self.bucket_params]

    def _broadcast_state(self, module: torch.nn.Module) -> None:
        """Algorithm 1 starts every worker from the same x_0: rank 0's parameters (the
        fusion buffer, so every bucket at once) and module buffers (BatchNorm running statistics)
        are broadcast over the process group, as torch DDP does at construction.  Afterwards the
        buffers stay local to each worker (SESGD averages parameters only, Eq. 6)."""
        import torch.distributed as dist
        grp = self.engine.group
        src = dist.get_global_rank(grp, 0)
        with torch.no_grad():
            for t in self.engine.x_flat:
                dist.broadcast(t, src=src, group=grp)
            for buf in module.buffers():
                dist.broadcast(buf, src=src, group=grp)
        torch.cuda.synchronize(self.engine.device)

    # ------------------------------------------------------------------ per step
    def enable_graphs(self) -> None:
        """Device-resident iterations (SESGD_OPT_DEVICE_ITER): from now on begin_step advances the
        iteration ON THE DEVICE (sesgd_begin_iter_device, the groups evaluated on the GPU), so a
        whole training step -- begin_step, forward, backward with the hook-launched bucket syncs on
        the side stream, finish_step -- can be captured once with torch.cuda.graph and replayed for
        every iteration.  Continues from the current iteration; needs the warm-up steps (and, with
        static_graph, the hook trimming of the first step) done eagerly first, and no tensor (e.g.
        the last eager loss) may still hold an eager step's autograd graph when the capture starts
        -- its AccumulateGrad nodes are bound to the eager stream, which a capture cannot join."""
        self.engine.set_device_iter(True)

    def begin_step(self, t: Optional[int] = None) -> None:
        """Start iteration t: zero the gradient buffers, set the schedule of t (device-resident
        iterations: the next iteration, on the device; t is ignored)."""
        self.t = self.t if t is None else t
        for g in self.engine.g_flat:
            g.zero_()
        if getattr(self.engine, "device_iter", False):
            self.engine.begin_iter_device(C.ITER_NEXT, torch.cuda.current_stream(self.engine.device))
        else:
            self.engine.begin_iter(self.t)
        self.ready.reset(self._hooked)
        self.launched_in_backward = 0  # buckets whose sync was enqueued from a gradient hook
        self._order = []

    def _launch(self, buckets) -> None:
        for b in buckets:  # in bucket order (BucketReadiness)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self.side.wait_event(ev)
            self.engine.sync_step(b, self.lr, self.momentum, self.side)

    def _on_grad(self, p: torch.Tensor) -> None:
        self._order.append(p)
        self._launch(self.ready.arrive(self.bucket_of[id(p)]))
        self.launched_in_backward = self.ready.next

    def finish_step(self) -> None:
        """After backward: sync every remaining bucket, then order the compute stream after the
        side stream (the next forward reads the updated parameters)."""
        self._launch(self.ready.force_all() if not self.overlap else self.ready.release())
        if not self.ready.done():
            raise RuntimeError("some gradients never arrived; every parameter must receive a gradient")
        self.done_event.record(self.side)
        torch.cuda.current_stream().wait_event(self.done_event)
        self.t += 1
        if self.static_graph and self.overlap and len(self._hooks) == len(self.params):
            self._trim_hooks()

    def _trim_hooks(self) -> None:
        last = {}
        for p in self._order:  # firing order of the step just finished
            last[self.bucket_of[id(p)]] = id(p)
        keep = set(last.values())
        for pid in [k for k in self._hooks if k not in keep]:
            self._hooks.pop(pid).remove()
        self._hooked = [1] * len(self.bucket_params)

    def close(self) -> None:
        for h in self._hooks.values():
            h.remove()
        self._hooks = {}
        if self._own_engine:
            self.engine.close()

"""SESGDEngine: owns the per-worker fp32 buckets as torch tensors and drives libsesgd.

PyTorch is used only for device memory, streams and process groups (symmetric
memory for the peer-visible workspace); all arithmetic runs in libsesgd's kernels.

Layout in HBM: per local worker one flat tensor per
array (x, v, g), buckets packed back to back at 64-float (256 B) aligned offsets,
so every bucket is a 16-byte-aligned view (128-bit vector path) and a model's
parameters/gradients can be views into the same storage (fusion buffer, no pack copy).
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import sesgd as C


def _aligned_offsets(sizes: Sequence[int], align: int = 64):
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += (int(s) + align - 1) // align * align
    return offs, max(o, align)


class SESGDEngine:
    def __init__(self, n: int, group_size: int, bucket_sizes: Sequence[int], *, seed: int = 42,
                 device: Optional[int] = None, mode: int = C.MODE_PARAM_AVG,
                 rank: int = 0, world: int = 1, process_group=None, path: int = C.PATH_AUTO,
                 grid: int = 0, timeout_ms: int = 20000, hop_delay_ns: int = 0,
                 p2p_variant: int = -1, discard: int = 1, options: Optional[dict] = None,
                 weight_decay: float = 0.0, loopback: bool = False, manual_peers: bool = False,
                 share_x_with: Optional["SESGDEngine"] = None):
        if n % world != 0:
            raise ValueError("n must be a multiple of the number of ranks")
        self.n, self.m, self.seed = n, group_size, seed
        self.path = path
        self.rank, self.world = rank, world
        self.r = n // world
        self.local_workers = list(range(rank * self.r, (rank + 1) * self.r))
        self.worker_rank = [i // self.r for i in range(n)]
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.bucket_sizes = [int(s) for s in bucket_sizes]
        self.ctx = C.sesgd_init(n, group_size, seed)
        C.sesgd_set_option(self.ctx, C.OPT_MODE, mode)
        C.sesgd_set_option(self.ctx, C.OPT_PATH, path)
        C.sesgd_set_option(self.ctx, C.OPT_TIMEOUT_MS, timeout_ms)
        C.sesgd_set_option(self.ctx, C.OPT_HOP_DELAY_NS, hop_delay_ns)
        if grid:
            C.sesgd_set_option(self.ctx, C.OPT_GRID, grid)
        if p2p_variant >= 0:
            C.sesgd_set_option(self.ctx, C.OPT_P2P_VARIANT, p2p_variant)
        C.sesgd_set_option(self.ctx, C.OPT_DISCARD, discard)
        for opt, val in (options or {}).items():  # extra SESGD_OPT_* (before the layout freezes)
            C.sesgd_set_option(self.ctx, opt, val)
        self.loopback = bool(loopback and world > 1)
        self.stream = None  # loopback: this virtual rank's own stream (set below)
        if self.loopback:  # `world` virtual ranks share this GPU: each sizes its grids for SMs / world
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            C.sesgd_set_option(self.ctx, C.OPT_SM_BUDGET, max(1, sms // world))
        if weight_decay:
            C.sesgd_set_weight_decay(self.ctx, weight_decay)
        C.sesgd_attach(self.ctx, self.device.index, self.local_workers)

        self.offsets, total = _aligned_offsets(self.bucket_sizes)
        mk = lambda: torch.zeros(total, dtype=torch.float32, device=self.device)  # noqa: E731
        # share_x_with: the final-average context (Alg.1's last line) works on another engine's
        # parameters, with its own zero momentum / gradient scratch
        self.x_flat = list(share_x_with.x_flat) if share_x_with is not None else [mk() for _ in range(self.r)]
        self.v_flat = [mk() for _ in range(self.r)]
        self.g_flat = [mk() for _ in range(self.r)]
        for b, numel in enumerate(self.bucket_sizes):
            C.sesgd_register_bucket(self.ctx, b, numel,
                                    [t.data_ptr() + 4 * self.offsets[b] for t in self.x_flat],
                                    [t.data_ptr() + 4 * self.offsets[b] for t in self.v_flat],
                                    [t.data_ptr() + 4 * self.offsets[b] for t in self.g_flat])
        self.workspace = None
        if self.loopback:  # a private workspace; LoopbackGroup attaches the virtual ranks to each other
            nbytes = C.sesgd_workspace_bytes(self.ctx)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            C.sesgd_workspace_prepare(self.ctx, self.workspace.data_ptr())
            self.stream = torch.cuda.Stream(device=self.device)
        elif world > 1 and manual_peers:
            # the caller maps the peers' workspaces itself (e.g. CUDA IPC, tools/ipc_pair.py) and
            # calls attach_peers(pointers): no process group, no NCCL
            nbytes = C.sesgd_workspace_bytes(self.ctx)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            C.sesgd_workspace_prepare(self.ctx, self.workspace.data_ptr())
        elif world > 1:
            self._attach_peers(process_group)
        elif path == C.PATH_ONESHOT:
            # single GPU through the one-shot kernel (profiling / tests): a private workspace
            nbytes = C.sesgd_workspace_bytes(self.ctx)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            C.sesgd_workspace_prepare(self.ctx, self.workspace.data_ptr())
            C.sesgd_attach_peers(self.ctx, 1, 0, [self.workspace.data_ptr()], self.worker_rank)

    # -------------------------------------------------------------- multi-GPU
    def _attach_peers(self, process_group):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        group = process_group or dist.group.WORLD
        self.group = group
        nbytes = C.sesgd_workspace_bytes(self.ctx)
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            try:
                symm_mem.enable_symm_mem_for_group(group.group_name)
            except Exception:  # already enabled / not needed in this torch
                pass
        self.workspace = symm_mem.empty(nbytes, dtype=torch.uint8, device=self.device)
        C.sesgd_workspace_prepare(self.ctx, self.workspace.data_ptr())
        self._symm = symm_mem.rendezvous(self.workspace, group)
        dist.barrier(group=group)
        ptrs = list(self._symm.buffer_ptrs)
        C.sesgd_attach_peers(self.ctx, self.world, self.rank, ptrs, self.worker_rank)
        if self.path == C.PATH_NVLS:  # NVLink SHARP: the multicast mapping of the same workspace
            mc = int(self._symm.multicast_ptr)
            if not mc:
                raise RuntimeError("SESGD_PATH_NVLS needs NVSwitch multicast (no multicast_ptr)")
            C.sesgd_attach_multicast(self.ctx, mc)
        dist.barrier(group=group)

    def attach_peers(self, ptrs) -> None:
        """manual_peers: every rank's workspace pointer, mapped in this process"""
        C.sesgd_attach_peers(self.ctx, self.world, self.rank, list(ptrs), self.worker_rank)

    # -------------------------------------------------------------- views
    def view(self, flat: torch.Tensor, b: int) -> torch.Tensor:
        o = self.offsets[b]
        return flat[o:o + self.bucket_sizes[b]]

    def x(self, slot: int, b: int) -> torch.Tensor:
        return self.view(self.x_flat[slot], b)

    def v(self, slot: int, b: int) -> torch.Tensor:
        return self.view(self.v_flat[slot], b)

    def g(self, slot: int, b: int) -> torch.Tensor:
        return self.view(self.g_flat[slot], b)

    # -------------------------------------------------------------- hot path
    def default_stream(self) -> torch.cuda.Stream:
        """the stream calls without an explicit one use: loopback virtual ranks each have their own
        (their persistent grids must run concurrently), otherwise torch's current stream"""
        return self.stream if self.stream is not None else torch.cuda.current_stream(self.device)

    def begin_iter(self, t: int) -> None:
        C.sesgd_begin_iter(self.ctx, t)

    # -------------------------------------------------------------- device-resident iterations
    def set_device_iter(self, on: bool = True) -> None:
        """SESGD_OPT_DEVICE_ITER: the iteration t, its groups (evaluated on the GPU from the shared
        seed) and the exchange call history live in device memory, so one captured CUDA
        graph replays every iteration.  Synchronous switch; off copies the state back."""
        C.sesgd_set_option(self.ctx, C.OPT_DEVICE_ITER, int(on))
        self.device_iter = bool(on)

    def begin_iter_device(self, t: int = C.ITER_NEXT, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else self.default_stream()
        C.sesgd_begin_iter_device(self.ctx, t, s.cuda_stream)

    def t_device_ptr(self) -> int:
        """device address of the int64 iteration counter (for t-dependent kernels in the graph)"""
        return C.sesgd_device_iter_ptr(self.ctx)

    def enqueue_iteration(self, lr: float, momentum: float, produce=None, fused: bool = True,
                          stream: Optional[torch.cuda.Stream] = None) -> None:
        """device-iteration mode: [next iteration on the device, produce(engine, stream) (e.g. the
        gradient fill reading t_device_ptr()), the sync launch(es)] on one stream"""
        s = stream if stream is not None else self.default_stream()
        self.begin_iter_device(C.ITER_NEXT, s)
        if produce is not None:
            produce(self, s)
        if fused:
            self.sync_all(lr, momentum, s)
        else:
            for b in range(len(self.bucket_sizes)):
                self.sync_step(b, lr, momentum, s)

    def capture_iteration(self, lr: float, momentum: float, produce=None, fused: bool = True):
        """one iteration (enqueue_iteration) captured ONCE into a CUDA graph; every replay
        (replay_iteration) runs the next iteration -- Algorithm 1's loop body with no
        host work per iteration.  Captured on this engine's own stream (loopback) or a side stream"""
        if not getattr(self, "device_iter", False):
            raise RuntimeError("capture_iteration needs set_device_iter(True)")
        if self.stream is not None:
            s = self.stream
        else:
            if getattr(self, "_capture_stream", None) is None:
                self._capture_stream = torch.cuda.Stream(device=self.device)
            s = self._capture_stream
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.enqueue_iteration(lr, momentum, produce, fused, s)
        return g

    def replay_iteration(self, g) -> None:
        """one replay of a captured iteration on this engine's default stream"""
        with torch.cuda.stream(self.default_stream()):
            g.replay()

    def sync_step(self, b: int, lr: float, momentum: float, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else self.default_stream()
        C.sesgd_sync_step(self.ctx, b, lr, momentum, s.cuda_stream)

    def sync_all(self, lr: float, momentum: float, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else self.default_stream()
        C.sesgd_sync_all(self.ctx, lr, momentum, s.cuda_stream)

    def step(self, t: int, lr: float, momentum: float, stream: Optional[torch.cuda.Stream] = None,
             fused: bool = True):
        """One SESGD iteration over every bucket (Alg.1 lines 3-11 for all local workers):
        one sesgd_sync_all call (fused), or one sesgd_sync_step per bucket."""
        if getattr(self, "device_iter", False):
            self.begin_iter_device(t, stream)
        else:
            self.begin_iter(t)
        if fused:
            self.sync_all(lr, momentum, stream)
        else:
            for b in range(len(self.bucket_sizes)):
                self.sync_step(b, lr, momentum, stream)

    def step_host(self, t: int, lr: float, momentum: float, g_host, x_host,
                  stream: Optional[torch.cuda.Stream] = None, pipelined: bool = True):
        """End-to-end through host buffers: g_host[b][slot] -> device, sync, device x ->
        x_host[b][slot]; pipelined (sesgd_sync_all_host: H2D / kernels / D2H of different
        buckets overlap) or one sesgd_sync_step_host per bucket."""
        s = stream if stream is not None else self.default_stream()
        self.begin_iter(t)
        if pipelined:
            C.sesgd_sync_all_host(self.ctx, lr, momentum, [h.data_ptr() for hb in g_host for h in hb],
                                  [h.data_ptr() for hb in x_host for h in hb], s.cuda_stream)
            return
        for b in range(len(self.bucket_sizes)):
            C.sesgd_sync_step_host(self.ctx, b, lr, momentum, [h.data_ptr() for h in g_host[b]],
                                   [h.data_ptr() for h in x_host[b]], s.cuda_stream)

    def average_engine(self, process_group=None) -> "SESGDEngine":
        """the final-average context: group_size = n over this engine's parameters, two-shot
        path (created on first use; every rank must call it)"""
        if getattr(self, "_avg", None) is None:
            self._avg = SESGDEngine(self.n, self.n, self.bucket_sizes, seed=self.seed, device=self.device.index,
                                    rank=self.rank, world=self.world, path=C.PATH_TWOSHOT,
                                    process_group=process_group or getattr(self, "group", None),
                                    loopback=self.loopback, share_x_with=self)
        return self._avg

    def global_average(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Algorithm 1's last line: every worker's parameters become the mean over all n
        workers (ascending fold, one division by n).  One GPU: K8 over the resident rows.  Several
        GPUs: one SESGD exchange with group_size = n through the two-shot NVLink kernel (K4 / K4W)
        on a context whose momentum and gradient are zero scratch and lr = 0, so x_hat = x exactly
        and the group mean is the global mean -- 2(n-1)/n x 4 B per element over NVLink instead of
        all-gathering (n-1) x 4 B."""
        if self.loopback:
            raise RuntimeError("loopback virtual ranks: use LoopbackGroup.global_average()")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        nb = len(self.bucket_sizes)
        if self.world == 1:
            for b in range(nb):
                C.sesgd_global_average(self.ctx, b, self.n, None, s.cuda_stream)
            return
        self.average_engine().step(0, 0.0, 0.0, s)

    def _gathered_rows(self, stream):
        """every rank's parameters, all-gathered (data movement only): [n, total] on this GPU"""
        import torch.distributed as dist
        with torch.cuda.stream(stream):
            local = torch.stack(self.x_flat)  # [r, total]
            gathered = torch.empty((self.world,) + tuple(local.shape), dtype=local.dtype, device=self.device)
            dist.all_gather_into_tensor(gathered, local, group=self.group)
        return gathered.view(self.n, -1)  # worker w = rank w // r, slot w % r: ascending id

    def consensus(self, stream: Optional[torch.cuda.Stream] = None):
        """Consistency of the workers' parameters (K9): (sum over workers and elements of
        (x_i - xbar)^2, max |x_i - xbar|), binary64."""
        if self.loopback:
            raise RuntimeError("loopback virtual ranks: use LoopbackGroup.consensus()")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        out = torch.zeros(2, dtype=torch.float64, device=self.device)
        rows = None if self.world == 1 else self._gathered_rows(s)
        for b in range(len(self.bucket_sizes)):
            ptrs = None if rows is None else [rows[w].data_ptr() + 4 * self.offsets[b] for w in range(self.n)]
            C.sesgd_consensus(self.ctx, b, self.n, out.data_ptr(), ptrs, s.cuda_stream)
        s.synchronize()
        return float(out[0]), float(out[1])

    def groups(self, t: int):
        return C.sesgd_groups(self.ctx, t, self.n)

    def stats(self, b: int) -> dict:
        return C.sesgd_get_stats(self.ctx, b)

    def poll(self) -> None:
        C.sesgd_poll(self.ctx)

    def measure_hop(self, peer_rank: int, iters: int = 5000, initiator: Optional[bool] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> None:
        """K7 ping-pong with `peer_rank` through the workspaces (both ranks call it concurrently);
        the one-way hop appears in stats()["hop_ns"] once the stream completes"""
        s = stream if stream is not None else self.default_stream()
        init = self.rank < peer_rank if initiator is None else initiator
        C.sesgd_measure_hop(self.ctx, peer_rank, iters, init, s.cuda_stream)

    def close(self) -> None:
        if getattr(self, "_avg", None) is not None:
            self._avg.close()
            self._avg = None
        if self.ctx is not None:
            C.sesgd_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """`world` virtual ranks on ONE GPU (SESGD_OPT_SM_BUDGET): every rank is an SESGDEngine with its
    own context, buffers, workspace and stream, attached to the others' workspaces through
    sesgd_attach_peers exactly as NVLink peers are -- so the multi-GPU kernels (K3 one-shot, K4
    two-shot, K5 ring) with their flags, stage / receive slots and reuse guards run, and are
    parity-tested, on a single B200.  Peer traffic goes through local HBM instead of NVLink, so
    loopback timings are not NVLink numbers.  Worker w lives on virtual rank w // (n / world)."""

    def __init__(self, world: int, n: int, group_size: int, bucket_sizes: Sequence[int], **kw):
        if world < 2:
            raise ValueError("a loopback group needs >= 2 virtual ranks")
        self.world = world
        self.engines = [SESGDEngine(n, group_size, bucket_sizes, rank=r, world=world, loopback=True, **kw)
                        for r in range(world)]
        ptrs = [e.workspace.data_ptr() for e in self.engines]
        torch.cuda.synchronize(self.engines[0].device)
        for e in self.engines:
            C.sesgd_attach_peers(e.ctx, world, e.rank, ptrs, e.worker_rank)
            e._siblings = self.engines

    def __getitem__(self, r: int) -> SESGDEngine:
        return self.engines[r]

    def __iter__(self):
        return iter(self.engines)

    def step(self, t: int, lr: float, momentum: float, fused: bool = True) -> None:
        """one iteration on every virtual rank: each enqueues its launch(es) on its own stream, so
        the R persistent grids run concurrently and exchange through each other's workspaces"""
        for e in self.engines:
            e.step(t, lr, momentum, fused=fused)

    def set_device_iter(self, on: bool = True) -> None:
        for e in self.engines:
            e.set_device_iter(on)

    def capture_iteration(self, lr: float, momentum: float, produce=None, fused: bool = True):
        """one CUDA graph per virtual rank (each captured on its own stream); replay() runs them
        concurrently, one iteration per replay"""
        return [e.capture_iteration(lr, momentum, produce, fused) for e in self.engines]

    def replay(self, graphs) -> None:
        for e, g in zip(self.engines, graphs):
            e.replay_iteration(g)

    def step_pair(self, t: int, lr: float, momentum: float) -> None:
        """measurement harness (two virtual ranks, K4W): both ranks' iteration as ONE kernel launch
        (sesgd_sync_all_pair) on rank 0's stream, so ncu can capture the exchange"""
        if self.world != 2:
            raise ValueError("the pair harness needs exactly two virtual ranks")
        e0, e1 = self.engines
        e0.begin_iter(t)
        e1.begin_iter(t)
        e0.stream.wait_stream(e1.stream)
        C.sesgd_sync_all_pair(e0.ctx, e1.ctx, lr, momentum, e0.stream.cuda_stream)
        e1.stream.wait_stream(e0.stream)

    def synchronize(self) -> None:
        for e in self.engines:
            e.stream.synchronize()

    def _gather(self):
        """every virtual rank's parameters after all queued work: [n, total] (data movement only)"""
        self.synchronize()
        return torch.cat([torch.stack(e.x_flat) for e in self.engines])

    def global_average(self) -> None:
        """Algorithm 1's last line on every virtual rank: one exchange with group_size = n
        through the two-shot kernel on zero-momentum contexts (as SESGDEngine.global_average)"""
        self.synchronize()
        if getattr(self, "_avg", None) is None:
            e0 = self.engines[0]
            self._avg = [SESGDEngine(e.n, e.n, e.bucket_sizes, seed=e.seed, device=e.device.index, rank=e.rank,
                                     world=e.world, path=C.PATH_TWOSHOT, loopback=True, share_x_with=e,
                                     timeout_ms=10000)
                         for e in self.engines]
            ptrs = [a.workspace.data_ptr() for a in self._avg]
            torch.cuda.synchronize(e0.device)
            for a in self._avg:
                C.sesgd_attach_peers(a.ctx, self.world, a.rank, ptrs, a.worker_rank)
        for a in self._avg:
            a.step(0, 0.0, 0.0)
        for a in self._avg:
            a.stream.synchronize()
        for a in self._avg:
            a.poll()

    def consensus(self):
        """K9 over the gathered rows, on virtual rank 0"""
        rows = self._gather()
        e = self.engines[0]
        out = torch.zeros(2, dtype=torch.float64, device=e.device)
        for b in range(len(e.bucket_sizes)):
            ptrs = [rows[w].data_ptr() + 4 * e.offsets[b] for w in range(e.n)]
            C.sesgd_consensus(e.ctx, b, e.n, out.data_ptr(), ptrs, e.stream.cuda_stream)
        e.stream.synchronize()
        return float(out[0]), float(out[1])

    def poll(self) -> None:
        for e in self.engines:
            e.poll()

    def close(self) -> None:
        for a in getattr(self, "_avg", None) or []:
            a.close()
        self._avg = None
        for e in self.engines:
            e.close()

"""World-size-2 gloo test of the decentralised schedule (CPU).

The paper avoids "extra message exchange" by seeding the same pseudo-random
algorithm on every worker.  Two processes each compute the schedule
through libsesgd on their own; gathering the results must show identical
partitions, and the worker -> rank placement used by the multi-GPU path must
put every worker on exactly one rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch
    from paper_2007_00433_b200 import sesgd as C
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, m, T = 16, 4, 64
    ctx = C.sesgd_init(n, m, 42)
    perms = np.stack([C.sesgd_groups(ctx, t, n)[0] for t in range(T)])
    C.sesgd_destroy(ctx)
    mine = torch.from_numpy(perms.astype(np.int64))
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    r = n // world
    local = torch.tensor(list(range(rank * r, (rank + 1) * r)), dtype=torch.int64)
    all_local = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(all_local, local)
    if rank == 0:
        out_q.put(([g.numpy() for g in gathered], [a.numpy() for a in all_local]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_compute_identical_schedules():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, locals_ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(gathered[0], gathered[1])
    placed = np.sort(np.concatenate(locals_))
    assert np.array_equal(placed, np.arange(16))


def test_reference_arm_under_torchrun_two_ranks():
    """bench.py --impl reference launched like the driver's N = 2 run (torchrun, two ranks, CPU):
    rank 0 prints exactly one JSON line with impl = reference, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(root, "bench.py"),
           "--gpus", "2", "--impl", "reference", "--steps", "2", "--warmup", "1"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0

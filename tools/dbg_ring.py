import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2007_00433_b200 import sesgd as C
from paper_2007_00433_b200.engine import LoopbackGroup
from cuda.bindings import runtime as rt
R = int(sys.argv[1]); n = R; m = int(sys.argv[2])
buckets = [70001, 4099, 333]
grp = LoopbackGroup(R, n, m, buckets, seed=42, path=C.PATH_RING, timeout_ms=3000)
def dump(e):
    return C.sesgd_device_iter_read(e.ctx, n, m, len(buckets))
offs = np.concatenate([[0], np.cumsum(buckets)[:-1]])
for e in grp:
    for b, L in enumerate(buckets):
        synth.fill_x0_device(e.x(0, b).data_ptr(), L, int(offs[b]), e.stream.cuda_stream)
grp.set_device_iter(True)
mode = sys.argv[3]
def produce(e, s):
    tp = e.t_device_ptr()
    for b, L in enumerate(buckets):
        synth.fill_grad_device_at(e.g(0, b).data_ptr(), L, int(offs[b]), e.local_workers[0], tp, s.cuda_stream)
if mode == "sync":
    for e in grp:
        e.begin_iter_device(0)
    grp.synchronize()
    for e in grp:
        print("rank", e.rank, dump(e), "host groups", e.groups(0)[0].tolist(), flush=True)
    for e in grp:
        for b in range(len(buckets)):
            e.sync_step(b, 0.1, 0.9)
elif mode == "interleaved":
    for it in range(3):
        for e in grp:
            e.enqueue_iteration(0.1, 0.9, produce, True)
elif mode == "serial":
    for it in range(3):
        for e in grp:
            e.enqueue_iteration(0.1, 0.9, None, True)
            print(it, "rank", e.rank, dump(e), flush=True)
elif mode == "begin_first":
    for it in range(3):
        for e in grp:
            e.begin_iter_device(C.ITER_NEXT)
        for e in grp:
            e.sync_all(0.1, 0.9)
elif mode == "noproduce":
    for it in range(3):
        for e in grp:
            e.enqueue_iteration(0.1, 0.9, None, True)
grp.synchronize()
for e in grp:
    print("after", e.rank, dump(e), flush=True)
    try:
        e.poll(); print("ok", e.rank)
    except Exception as ex:
        print("ERR", e.rank, ex)

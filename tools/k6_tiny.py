"""One small SESGD run on cuda:0 through the resident kernel K6 (both modes, per-bucket and
fused launches, an odd bucket size for the vector tails), for tools/sanitize.sh."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2007_00433_b200 import sesgd as C  # noqa: E402
from paper_2007_00433_b200.engine import SESGDEngine  # noqa: E402

buckets = [20003, 7, 4099]
for mode in (C.MODE_PARAM_AVG, C.MODE_GRAD_AVG):
    eng = SESGDEngine(4, 2, buckets, seed=42, mode=mode)
    st = torch.cuda.current_stream().cuda_stream
    off = 0
    for b, L in enumerate(buckets):
        for s in range(eng.r):
            synth.fill_x0_device(eng.x(s, b).data_ptr(), L, off, st)
            synth.fill_grad_device(eng.g(s, b).data_ptr(), L, off, s, 0, st)
        off += L
    for t in range(3):
        eng.step(t, 0.1, 0.9, fused=bool(t % 2))
    torch.cuda.synchronize()
    eng.poll()
    eng.close()
print("k6_tiny ok")

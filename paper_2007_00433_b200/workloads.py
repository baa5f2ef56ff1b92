"""Synthetic workload shapes.

Per-parameter-tensor element counts of torchvision ResNet-50 and VGG-16 (random init;
only the SHAPES matter -- values come from synth/), in registration order, and the
DDP-style bucketing the paper's integration imitates ("imitating the PyTorch
DistributedDataParallel module"): reverse registration order, first bucket capped at
1 MiB, the rest at 25 MiB, a bucket closes once it reaches its cap.
"""
from __future__ import annotations

from typing import List, Sequence

RESNET50_TENSORS = (
    9408, 64, 64, 4096, 64, 64, 36864, 64, 64, 16384, 256, 256,
    16384, 256, 256, 16384, 64, 64, 36864, 64, 64, 16384, 256, 256,
    16384, 64, 64, 36864, 64, 64, 16384, 256, 256, 32768, 128, 128,
    147456, 128, 128, 65536, 512, 512, 131072, 512, 512, 65536, 128, 128,
    147456, 128, 128, 65536, 512, 512, 65536, 128, 128, 147456, 128, 128,
    65536, 512, 512, 65536, 128, 128, 147456, 128, 128, 65536, 512, 512,
    131072, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 524288, 1024, 1024,
    262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256,
    589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256,
    262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024,
    262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 524288, 512, 512,
    2359296, 512, 512, 1048576, 2048, 2048, 2097152, 2048, 2048, 1048576, 512, 512,
    2359296, 512, 512, 1048576, 2048, 2048, 1048576, 512, 512, 2359296, 512, 512,
    1048576, 2048, 2048, 2048000, 1000,
)

VGG16_TENSORS = (
    1728, 64, 36864, 64, 73728, 128, 147456, 128, 294912, 256, 589824, 256,
    589824, 256, 1179648, 512, 2359296, 512, 2359296, 512, 2359296, 512, 2359296, 512,
    2359296, 512, 102760448, 4096, 16777216, 4096, 4096000, 1000,
)


def ddp_buckets(tensor_sizes: Sequence[int], first_cap_bytes: int = 1 << 20,
                cap_bytes: int = 25 << 20, elem_bytes: int = 4) -> List[int]:
    caps = (first_cap_bytes // elem_bytes, cap_bytes // elem_bytes)
    out: List[int] = []
    cur = 0
    for s in reversed(tensor_sizes):
        cur += int(s)
        if cur >= caps[min(len(out), 1)]:
            out.append(cur)
            cur = 0
    if cur:
        out.append(cur)
    return out


# BASELINE.json configs[0]: 3 buckets summing to 2^20 with odd sizes (vector tails)
CONFIG1_BUCKETS = (699051, 262147, 87378)
RESNET50_BUCKETS = tuple(ddp_buckets(RESNET50_TENSORS))
VGG16_BUCKETS = tuple(ddp_buckets(VGG16_TENSORS))

WORKLOADS = {
    "config1": CONFIG1_BUCKETS,
    "resnet50": RESNET50_BUCKETS,
    "vgg16": VGG16_BUCKETS,
    "resnet50_per_layer": RESNET50_TENSORS,
}

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


def assign_buckets(tensor_sizes: Sequence[int], first_cap_bytes: int = 1 << 20,
                   cap_bytes: int = 25 << 20, elem_bytes: int = 4) -> List[List[int]]:
    """Tensor indices per bucket: reverse registration order, a bucket closes once it reaches
    its cap (first 1 MiB, the rest 25 MiB)."""
    caps = (first_cap_bytes // elem_bytes, cap_bytes // elem_bytes)
    out: List[List[int]] = []
    cur: List[int] = []
    total = 0
    for i in reversed(range(len(tensor_sizes))):
        cur.append(i)
        total += int(tensor_sizes[i])
        if total >= caps[min(len(out), 1)]:
            out.append(cur)
            cur, total = [], 0
    if cur:
        out.append(cur)
    return out


def ddp_buckets(tensor_sizes: Sequence[int], first_cap_bytes: int = 1 << 20,
                cap_bytes: int = 25 << 20, elem_bytes: int = 4) -> List[int]:
    """Elements per bucket of assign_buckets."""
    return [sum(int(tensor_sizes[i]) for i in b)
            for b in assign_buckets(tensor_sizes, first_cap_bytes, cap_bytes, elem_bytes)]


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

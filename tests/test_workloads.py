"""Host logic of the workload shapes and the DDP-style bucketing (CPU only)."""
import pytest
import torch

from paper_2007_00433_b200.workloads import (RESNET50_BUCKETS, RESNET50_TENSORS, VGG16_BUCKETS,
                                             VGG16_TENSORS, assign_buckets, ddp_buckets)


def test_tensor_lists_match_torchvision():
    tv = pytest.importorskip("torchvision")
    with torch.device("meta"):
        r50 = [p.numel() for p in tv.models.resnet50().parameters()]
        vgg = [p.numel() for p in tv.models.vgg16().parameters()]
    assert tuple(r50) == RESNET50_TENSORS
    assert tuple(vgg) == VGG16_TENSORS
    assert sum(r50) == 25_557_032 and sum(vgg) == 138_357_544


def test_resnet50_ddp_buckets():
    # reverse order: fc (2,049,000 = 2048*1000 + 1000) alone passes the 1 MiB cap
    assert RESNET50_BUCKETS == (2049000, 7875584, 6563840, 6637568, 2431040)
    assert VGG16_BUCKETS[0] == 4097000 and sum(VGG16_BUCKETS) == 138_357_544


@pytest.mark.parametrize("first,cap", [(1 << 20, 25 << 20), (16 << 10, 256 << 10), (4, 4), (1 << 40, 1 << 40)])
def test_assign_buckets_partition(first, cap):
    sizes = RESNET50_TENSORS
    bk = assign_buckets(sizes, first, cap)
    flat = [i for b in bk for i in b]
    assert flat == list(reversed(range(len(sizes))))  # every tensor once, reverse registration order
    caps = [first // 4] + [cap // 4] * (len(bk) - 1)
    for j, b in enumerate(bk):
        tot = sum(sizes[i] for i in b)
        assert tot >= caps[j] or j == len(bk) - 1                 # closes at its cap (last: remainder)
        assert tot - sizes[b[-1]] < caps[j]                       # ... and not later
    assert ddp_buckets(sizes, first, cap) == [sum(sizes[i] for i in b) for b in bk]


def test_ddp_wrapper_requires_one_worker_per_rank():
    from paper_2007_00433_b200.ddp import SESGDDataParallel
    with pytest.raises(ValueError):
        SESGDDataParallel(torch.nn.Linear(2, 2), 2, 2, lr=0.1, momentum=0.9, rank=0, world=1)


@pytest.mark.parametrize("sizes", [RESNET50_BUCKETS, VGG16_BUCKETS, [699051, 262147, 87378], [0, 1, 0, 7], []])
def test_fusion_buffer_offsets_are_256B_aligned_and_disjoint(sizes):
    """bucket b sits at round_up(sum of earlier sizes, 64 floats) -- every bucket
    256 B aligned (the 128-bit path always applies), buckets never overlap, the buffer holds all."""
    from paper_2007_00433_b200.engine import _aligned_offsets
    offs, total = _aligned_offsets(sizes)
    assert len(offs) == len(sizes)
    end = 0
    for o, s in zip(offs, sizes):
        assert o % 64 == 0 and o >= end and o - end < 64
        end = o + s
    assert total >= end and total % 64 == 0 and total - end < 64 + 64

"""B200-native hot path of Shuffle-Exchange SGD (arXiv 2007.00433).

``sesgd``   -- thin ctypes binding of libsesgd.so (include/sesgd.h), same call names.
``engine``  -- SESGDEngine: torch-owned fp32 buckets + multi-GPU workspace, drives libsesgd.
``workloads`` -- ResNet-50 / VGG-16 tensor shapes and DDP-style buckets.
"""
from . import sesgd, workloads  # noqa: F401
from .sesgd import *  # noqa: F401,F403

__all__ = ["sesgd", "workloads", "engine"]

"""B200-native 1-bit LAMB compression-stage path (arXiv 2104.06069).

The product is libbitlamb_b200.so (hand-written sm_100a kernels + the C-ABI of
include/bitlamb_b200.h).  `bitlamb` mirrors the reference's SimCluster /
Optimizer API over that ABI; `layouts` holds the synthetic BERT layer tables.
"""
from . import layouts  # noqa: F401

__all__ = ["layouts"]

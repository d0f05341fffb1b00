"""TCM-Serve's per-iteration modality-aware scheduling step (arxiv 2603.26498) on B200.

The product is libtcm.so (C ABI, include/tcm.h) with sm_100a kernels; `tcm` is its thin
ctypes binding and `sharding` the replica-sharding layer over torch.distributed.
"""
from . import tcm  # noqa: F401

__all__ = ["tcm"]

"""B200-native MG-GCN full-batch training step (arXiv 2110.08688) behind the reference's training API.

The product is libmggcn.so (CUDA sm_100a kernels + NCCL + host C++ partitioner) behind the C ABI in
include/mggcn.h; `rowgcn` mirrors the reference's (rowgcn) API on top of it.
"""
from . import rowgcn  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["rowgcn", "lib", "LIB_PATH"]

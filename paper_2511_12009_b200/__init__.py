"""B200-native N-Queens solution counter (arXiv 2511.12009 capabilities).

The counting path — folded frontier generation, the persistent sm_100a DFS kernel,
the intra-GPU work queue and count reduction, and the multi-GPU chunk scheduler — lives
in libnqb200.so behind the C ABI of include/nq_gpu.h. This package is its Python face:
`nqueens` mirrors the reference's C++ API (execute, execute_batch, generate, ...).
"""
from . import nqueens
from ._build import LIB_PATH, build

__all__ = ["nqueens", "build", "LIB_PATH"]

"""B200-native N-Queens solution counter (arXiv 2511.12009 capabilities).

The counting path — folded frontier generation, the persistent sm_100a DFS kernel,
the intra-GPU work queue and count reduction, and the multi-GPU chunk scheduler — lives
in libnqb200.so behind the C ABI of include/nq_gpu.h. This package is its Python face:
`nqueens` mirrors the reference's C++ API (execute, execute_batch, generate, ...).

`nqueens` is imported lazily so that `_build` can compile the library before anything
loads it; importing `nqueens` raises ImportError when libnqb200.so is missing.
"""
from ._build import LIB_PATH, build

__all__ = ["nqueens", "build", "LIB_PATH"]


def __getattr__(name):
    if name == "nqueens":
        import importlib
        return importlib.import_module(".nqueens", __name__)
    raise AttributeError(name)

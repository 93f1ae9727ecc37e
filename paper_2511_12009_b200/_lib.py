"""ctypes binding of libnqb200.so (the C ABI declared in include/nq_gpu.h).

The library is REQUIRED: there is no Python or CPU fallback for counting. Importing
this module loads the in-tree .so and raises if it is missing; a missing or
non-sm_100 GPU surfaces as NqError(NQ_ECUDA) from the first counting call.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB_PATH

NQ_OK = 0
NQ_ECUDA = -1
NQ_ECONFIG = -2
NQ_EOVERFLOW = -3
NQ_ECANCEL = -4
NQ_ECHECKPOINT = -5

LAYOUT_V4, LAYOUT_PLANES = 0, 1

VARIANT_ITERATIVE = 0
VARIANT_LASTROW = 1

# Packed 16-byte frontier record: row = placed_rows | multiplier << 8.
SUB_DTYPE = np.dtype([("cols", "<u4"), ("diag", "<u4"), ("antidiag", "<u4"), ("row", "<u4")])


class NqSub(ctypes.Structure):
    _fields_ = [("cols", ctypes.c_uint32), ("diag", ctypes.c_uint32),
                ("antidiag", ctypes.c_uint32), ("row", ctypes.c_uint32)]


class NqResult(ctypes.Structure):
    _fields_ = [("solutions", ctypes.c_uint64), ("raw_solutions", ctypes.c_uint64),
                ("nodes", ctypes.c_uint64), ("iterations", ctypes.c_uint64),
                ("subproblems", ctypes.c_uint64), ("kernel_ms", ctypes.c_double),
                ("h2d_ms", ctypes.c_double)]


NQ_LOG_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_char_p)


class NqSolveOpts(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("strategy", ctypes.c_int),
                ("worker_count", ctypes.c_int), ("weights", ctypes.POINTER(ctypes.c_double)),
                ("chunk", ctypes.c_uint64), ("n_devices", ctypes.c_int),
                ("devices", ctypes.POINTER(ctypes.c_int)), ("cancel", ctypes.POINTER(ctypes.c_int)),
                ("stack_depth", ctypes.c_int), ("config_name", ctypes.c_char_p),
                ("log", NQ_LOG_FN), ("log_user", ctypes.c_void_p),
                ("dispatch", ctypes.c_void_p)]


MAX_WORKERS = 64


class NqWorkerStats(ctypes.Structure):
    _fields_ = [("worker", ctypes.c_int), ("device", ctypes.c_int),
                ("assigned", ctypes.c_uint64), ("processed", ctypes.c_uint64),
                ("partial_sum", ctypes.c_uint64), ("nodes", ctypes.c_uint64),
                ("chunks", ctypes.c_uint64), ("elapsed_ms", ctypes.c_double),
                ("kernel_ms", ctypes.c_double), ("span_ms", ctypes.c_double),
                ("launches", ctypes.c_uint64)]


class NqReport(ctypes.Structure):
    _fields_ = [("total", ctypes.c_uint64), ("task_count", ctypes.c_uint64),
                ("nodes", ctypes.c_uint64), ("generation_ms", ctypes.c_double),
                ("calc_ms", ctypes.c_double), ("completed", ctypes.c_int),
                ("worker_count", ctypes.c_int), ("workers", NqWorkerStats * MAX_WORKERS)]


class NqCkptOpts(ctypes.Structure):
    _fields_ = [("path", ctypes.c_char_p), ("chunk", ctypes.c_uint64),
                ("flush_interval_s", ctypes.c_double), ("resume", ctypes.c_int),
                ("stop_after_s", ctypes.c_double)]


PARTITION_UNIFORM, PARTITION_WEIGHTED, PARTITION_STEALING, PARTITION_GUIDED, PARTITION_STRIDED = 0, 1, 2, 3, 4
LOG_GENERATION, LOG_START, LOG_FINISH, LOG_RESULT = 0, 1, 2, 3


class NqError(RuntimeError):
    """A non-zero status from the C ABI; .code is the NQ_E* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the counting path)")
    return ctypes.CDLL(LIB_PATH)


lib = _load()

_P = ctypes.POINTER
_u64 = ctypes.c_uint64
_sigs = {
    "nq_abi_version": (ctypes.c_int, []),
    "nq_last_error": (ctypes.c_char_p, []),
    "nq_device_count": (ctypes.c_int, [_P(ctypes.c_int)]),
    "nq_ctx_create": (ctypes.c_int, [ctypes.c_int, _P(ctypes.c_void_p)]),
    "nq_ctx_destroy": (None, [ctypes.c_void_p]),
    "nq_ctx_set_tuning": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "nq_ctx_set_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "nq_ctx_set_cancel": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "nq_ctx_set_balance": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "nq_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p, _u64, _P(NqResult)]),
    "nq_count_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, _u64, _P(NqResult)]),
    "nq_count_device_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_void_p, _u64]),
    "nq_collect": (ctypes.c_int, [ctypes.c_void_p, _P(NqResult)]),
    "nq_expand_device": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64, ctypes.c_int,
                                        ctypes.c_void_p, _u64, _P(_u64)]),
    "nq_count_expand": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, _u64, _P(NqResult)]),
    "nq_count_each": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, _u64, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    "nq_generate": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64, _P(_u64)]),
    "nq_generate_slice": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _u64, _u64, ctypes.c_void_p,
                                         _u64, _P(_u64)]),
    "nq_count_subproblems": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P(_u64)]),
    "nq_expand": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, _u64, ctypes.c_int, ctypes.c_void_p,
                                 _u64, _P(_u64)]),
    "nq_solve_batch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64,
                                      _P(NqSolveOpts), _P(NqReport)]),
    "nq_solve": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P(NqSolveOpts), _P(NqReport)]),
    "nq_solve_batch_expand": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64,
                                             _P(NqSolveOpts), _P(NqReport)]),
    "nq_solve_batch_device": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P(ctypes.c_void_p), _u64,
                                             _P(NqSolveOpts), _P(NqReport)]),
    "nq_dispatch_create": (ctypes.c_int, [ctypes.c_char_p, _u64, ctypes.c_int, _u64, ctypes.c_int,
                                          _P(ctypes.c_void_p)]),
    "nq_dispatch_attach": (ctypes.c_int, [ctypes.c_char_p, _P(ctypes.c_void_p)]),
    "nq_dispatch_close": (None, [ctypes.c_void_p, ctypes.c_int]),
    "nq_dispatch_take": (ctypes.c_int, [ctypes.c_void_p, _P(_u64), _P(_u64)]),
    "nq_dispatch_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "nq_dispatch_info": (ctypes.c_int, [ctypes.c_void_p, _P(_u64), _P(ctypes.c_int), _P(_u64),
                                        _P(ctypes.c_int)]),
    "nq_dispatch_post": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u64, _u64, _u64]),
    "nq_dispatch_sum": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _P(_u64), _P(_u64), _P(_u64)]),
    "nq_solve_checkpointed": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P(NqSolveOpts),
                                             _P(NqCkptOpts), _P(NqReport)]),
    "nq_checkpoint_info": (ctypes.c_int, [ctypes.c_char_p, _P(ctypes.c_int), _P(ctypes.c_int),
                                          _P(ctypes.c_int), _P(_u64), _P(_u64), _P(_u64)]),
    "nq_checkpoint_read": (ctypes.c_int, [ctypes.c_char_p, _P(ctypes.c_int), _P(ctypes.c_int),
                                          _P(_u64), _P(_u64)]),
    "nq_partition_uniform": (ctypes.c_int, [_u64, ctypes.c_int, _P(_u64)]),
    "nq_partition_weighted": (ctypes.c_int, [_u64, _P(ctypes.c_double), ctypes.c_int, _P(_u64)]),
    "nq_format_log": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _u64, ctypes.c_double,
                                     ctypes.c_char_p, _u64]),
    "nq_measure_int_peak": (ctypes.c_int, [ctypes.c_int, _P(ctypes.c_double),
                                           _P(ctypes.c_double)]),
}
for _name, (_res, _args) in _sigs.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_sigs)


def check(rc: int) -> None:
    if rc != NQ_OK:
        msg = lib.nq_last_error().decode(errors="replace")
        raise NqError(rc, msg)

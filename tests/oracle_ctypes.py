"""ctypes access to the CHECKERS under oracle/ (test infrastructure only).

  * oracle/_build/libnqoracle.so — the plain-C restatement (oracle/nq_oracle.c)
  * oracle/_ref/libnqref.so      — the reference headers compiled from
                                   /root/reference (oracle/ref_shim.cpp); optional

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load these.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "_build", "libnqoracle.so")
REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libnqref.so")
SUB_DTYPE = np.dtype([("cols", "<u4"), ("diag", "<u4"), ("antidiag", "<u4"), ("row", "<u4")])

_u64 = ctypes.c_uint64
_P = ctypes.POINTER


def build_oracle() -> None:
    """make -C oracle (the C restatement always; the reference build when its tree exists)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Oracle:
    """The C restatement of the reference counting path."""

    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            build_oracle()
        L = self.L = ctypes.CDLL(path)
        L.nqo_last_error.restype = ctypes.c_char_p
        L.nqo_count_recursive.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, _P(_u64)]
        L.nqo_count_iterative.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, _P(_u64),
                                          _P(ctypes.c_int)]
        L.nqo_count_lastrow.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, _P(_u64),
                                        _P(ctypes.c_int), _P(_u64)]
        L.nqo_generate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64, _P(_u64)]
        L.nqo_count_subproblems.argtypes = [ctypes.c_int, ctypes.c_int, _P(_u64)]
        L.nqo_aggregate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64, _P(_u64)]
        L.nqo_partition_uniform.argtypes = [_u64, ctypes.c_int, ctypes.c_void_p]
        L.nqo_partition_weighted.argtypes = [_u64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.nqo_solve_batch.argtypes = [ctypes.c_int, ctypes.c_void_p, _u64, ctypes.c_int, _u64,
                                      _P(_u64), _P(_u64), ctypes.c_void_p]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.nqo_last_error().decode())

    def count_recursive(self, n, cur, left, right) -> int:
        out = _u64()
        self._chk(self.L.nqo_count_recursive(n, cur, left, right, ctypes.byref(out)))
        return out.value

    def count_iterative(self, n, rec, depth=24):
        a = np.array([rec], dtype=SUB_DTYPE)
        c, h = _u64(), ctypes.c_int()
        self._chk(self.L.nqo_count_iterative(n, a.ctypes.data, depth, ctypes.byref(c), ctypes.byref(h)))
        return c.value, h.value

    def count_lastrow(self, n, rec, depth=24):
        a = np.array([rec], dtype=SUB_DTYPE)
        c, h, nd = _u64(), ctypes.c_int(), _u64()
        self._chk(self.L.nqo_count_lastrow(n, a.ctypes.data, depth, ctypes.byref(c), ctypes.byref(h),
                                           ctypes.byref(nd)))
        return c.value, h.value, nd.value

    def generate(self, n, r) -> np.ndarray:
        total = _u64()
        self._chk(self.L.nqo_generate(n, r, None, 0, ctypes.byref(total)))
        a = np.zeros(total.value, dtype=SUB_DTYPE)
        self._chk(self.L.nqo_generate(n, r, a.ctypes.data, total.value, ctypes.byref(total)))
        return a

    def count_subproblems(self, n, r) -> int:
        t = _u64()
        self._chk(self.L.nqo_count_subproblems(n, r, ctypes.byref(t)))
        return t.value

    def aggregate(self, subs: np.ndarray, counts) -> int:
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        t = _u64()
        self._chk(self.L.nqo_aggregate(subs.ctypes.data, c.ctypes.data, len(subs), ctypes.byref(t)))
        return t.value

    def partition_uniform(self, tasks, workers):
        buf = np.zeros(2 * max(workers, 1), dtype=np.uint64)
        self._chk(self.L.nqo_partition_uniform(tasks, workers, buf.ctypes.data))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(workers)]

    def partition_weighted(self, tasks, weights):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        buf = np.zeros(2 * max(len(w), 1), dtype=np.uint64)
        self._chk(self.L.nqo_partition_weighted(tasks, w.ctypes.data, len(w), buf.ctypes.data))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(len(w))]

    def solve_batch(self, n, subs: np.ndarray, threads=None, chunk=64, per_sub=False):
        threads = threads or os.cpu_count() or 1
        tot, nodes = _u64(), _u64()
        ps = np.zeros(len(subs), dtype=np.uint64) if per_sub else None
        self._chk(self.L.nqo_solve_batch(n, subs.ctypes.data if len(subs) else None, len(subs),
                                         threads, chunk, ctypes.byref(tot), ctypes.byref(nodes),
                                         ps.ctypes.data if per_sub else None))
        return (tot.value, nodes.value, ps) if per_sub else (tot.value, nodes.value)


class Reference:
    """The unmodified reference headers compiled into oracle/_ref/libnqref.so."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = ctypes.CDLL(path)
        L.nqref_last_error.restype = ctypes.c_char_p
        L.nqref_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                  _P(_u64), _P(ctypes.c_int)]
        L.nqref_generate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64, _P(_u64)]
        L.nqref_count_subproblems.argtypes = [ctypes.c_int, ctypes.c_int, _P(_u64)]
        L.nqref_generate_slice.argtypes = [ctypes.c_int, ctypes.c_int, _u64, _u64, ctypes.c_void_p,
                                           _u64, _P(_u64)]
        L.nqref_conflict_degree.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                            _u64, ctypes.c_int, ctypes.c_int, _P(ctypes.c_int),
                                            _P(ctypes.c_int)]
        L.nqref_write_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _u64, _P(_u64)]
        L.nqref_aggregate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64, _P(_u64)]
        L.nqref_partition.argtypes = [ctypes.c_int, _u64, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_void_p]
        L.nqref_execute_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _u64,
                                          ctypes.c_int, ctypes.c_int, _u64, ctypes.c_int,
                                          ctypes.c_int, _P(_u64), _P(ctypes.c_double), _P(_u64)]
        L.nqref_execute.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64,
                                    ctypes.c_int, ctypes.c_int, _P(_u64), _P(ctypes.c_double),
                                    _P(ctypes.c_double), _P(_u64)]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.nqref_last_error().decode())

    def count(self, variant, n, rec, config_index=0):
        """variant: 0 iterative, 1 lastrow, 2 recursive."""
        a = np.array([rec], dtype=SUB_DTYPE)
        c, h = _u64(), ctypes.c_int()
        self._chk(self.L.nqref_count(variant, n, a.ctypes.data, config_index, ctypes.byref(c),
                                     ctypes.byref(h)))
        return c.value, h.value

    def generate(self, n, r) -> np.ndarray:
        total = _u64()
        self._chk(self.L.nqref_generate(n, r, None, 0, ctypes.byref(total)))
        a = np.zeros(total.value, dtype=SUB_DTYPE)
        self._chk(self.L.nqref_generate(n, r, a.ctypes.data, total.value, ctypes.byref(total)))
        return a

    def count_subproblems(self, n, r) -> int:
        t = _u64()
        self._chk(self.L.nqref_count_subproblems(n, r, ctypes.byref(t)))
        return t.value

    def generate_slice(self, n, r, stride, offset=0) -> np.ndarray:
        """Records i ≡ offset (mod stride) of the reference's own stream."""
        total = _u64()
        self._chk(self.L.nqref_generate_slice(n, r, stride, offset, None, 0, ctypes.byref(total)))
        a = np.zeros(total.value, dtype=SUB_DTYPE)
        self._chk(self.L.nqref_generate_slice(n, r, stride, offset, a.ctypes.data, total.value,
                                              ctypes.byref(total)))
        return a

    def conflict_degree(self, addresses, width, full_warp=False, banks=32, word=4, warp=32):
        """bankmodel.hpp:62-99 -> (transactions, max_degree)."""
        a = np.ascontiguousarray(addresses, dtype=np.uint64)
        t, d = ctypes.c_int(), ctypes.c_int()
        self._chk(self.L.nqref_conflict_degree(banks, word, warp, a.ctypes.data if len(a) else None,
                                               len(a), width, 1 if full_warp else 0,
                                               ctypes.byref(t), ctypes.byref(d)))
        return t.value, d.value

    def write_batch(self, n, r) -> str:
        ln = _u64()
        self._chk(self.L.nqref_write_batch(n, r, None, 0, ctypes.byref(ln)))
        buf = ctypes.create_string_buffer(ln.value + 1)
        self._chk(self.L.nqref_write_batch(n, r, buf, ln.value, ctypes.byref(ln)))
        return buf.raw[: ln.value].decode()

    def execute_batch(self, n, r, subs: np.ndarray, workers, chunk=64, strategy=2, variant=1,
                      config_index=0):
        tot, ms, proc = _u64(), ctypes.c_double(), _u64()
        self._chk(self.L.nqref_execute_batch(n, r, subs.ctypes.data if len(subs) else None,
                                             len(subs), strategy, workers, chunk, variant,
                                             config_index, ctypes.byref(tot), ctypes.byref(ms),
                                             ctypes.byref(proc)))
        return tot.value, ms.value, proc.value


def reference_available() -> bool:
    return os.path.exists(REF_LIB)

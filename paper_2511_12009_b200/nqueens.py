"""Python mirror of the reference's nqueens API for the counting path.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/nqueens/{bitboard,errors,stack_config,solver,subproblems,
scheduler}.hpp, so tests read like the reference's doctest suite. Every counting call
runs the sm_100a kernels of libnqb200.so through its C ABI (include/nq_gpu.h); the
frontier is produced by the library's multi-threaded C++ generator.

Exceptions: ConfigError (~ nqueens::config_error), OverflowError (~ std::overflow_error,
Python's builtin), RuntimeError (~ std::runtime_error, worker failures).
"""
from __future__ import annotations

import ctypes
import enum
import io
import threading
from dataclasses import dataclass, field
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import SUB_DTYPE, NqError, check, lib

MASK64 = (1 << 64) - 1
kMaxBoard = 32
kQueens27Reference = 234907967154122528  # subproblems.hpp:28


class ConfigError(ValueError):
    """nqueens::config_error (errors.hpp:10-13)."""


config_error = ConfigError


class CheckpointError(RuntimeError):
    """nqueens::checkpoint_error (errors.hpp:16-19): unreadable, corrupt or foreign file."""


checkpoint_error = CheckpointError


def _raise(err: NqError):
    if err.code == _lib.NQ_ECONFIG:
        raise ConfigError(str(err)) from None
    if err.code == _lib.NQ_EOVERFLOW:
        raise OverflowError(str(err)) from None
    if err.code == _lib.NQ_ECHECKPOINT:
        raise CheckpointError(str(err)) from None
    raise RuntimeError(str(err)) from None


def _call(rc: int) -> None:
    try:
        check(rc)
    except NqError as e:
        _raise(e)


# ---- errors.hpp:23-35 ---------------------------------------------------------------------
def checked_add(a: int, b: int) -> int:
    r = a + b
    if r > MASK64:
        raise OverflowError("solution count overflows 64 bits")
    return r


def checked_mul(a: int, b: int) -> int:
    r = a * b
    if r > MASK64:
        raise OverflowError("solution count overflows 64 bits")
    return r


# ---- bitboard.hpp (host-side helpers; the device has its own PTX) --------------------------
def board_mask(n: int) -> int:
    return 0xFFFFFFFF if n >= 32 else (1 << n) - 1


def valid_positions(cur: int, left: int, right: int, n: int) -> int:
    return board_mask(n) & ~(cur | left | right) & 0xFFFFFFFF


def lowest_set_bit(mask: int) -> int:
    assert mask != 0
    return mask & (-mask) & 0xFFFFFFFF


@dataclass(frozen=True)
class PlacementState:
    cur: int
    left: int
    right: int


def apply_placement(cur: int, left: int, right: int, p: int) -> PlacementState:
    return PlacementState(cur | p, ((left | p) << 1) & 0xFFFFFFFF, (right | p) >> 1)


# ---- stack_config.hpp ----------------------------------------------------------------------
@dataclass(frozen=True)
class StackConfig:
    name: str
    block_size: int = 128
    stack_words: int = 96
    pre_rows_reference: int = 6
    last_row_opt: bool = False

    def max_depth(self) -> int:
        return self.stack_words // 4

    def max_n(self) -> int:
        return self.max_depth() + self.pre_rows_reference + (1 if self.last_row_opt else 0)


builtin_configs = (
    StackConfig("config1", 128, 96),
    StackConfig("config2", 160, 76),
    StackConfig("config3", 192, 64),
    StackConfig("config4", 256, 48),
    StackConfig("config5", 512, 24),
)


def find_config(name: str) -> Optional[StackConfig]:
    return next((c for c in builtin_configs if c.name == name), None)


def required_depth(n: int, placed_rows: int, last_row: bool) -> int:
    return n - placed_rows - (1 if last_row else 0)


def smallest_sufficient_config(n: int, placed_rows: int, last_row: bool) -> Optional[StackConfig]:
    need = required_depth(n, placed_rows, last_row)
    fits = [c for c in builtin_configs if c.max_depth() >= need]
    return min(fits, key=lambda c: c.max_depth()) if fits else None


def require_feasible(cfg: StackConfig, n: int, placed_rows: int, last_row: bool) -> None:
    need = required_depth(n, placed_rows, last_row)
    if need <= cfg.max_depth():
        return
    msg = (f"stack config '{cfg.name}' supports depth {cfg.max_depth()} but n={n}, "
           f"pre_rows={placed_rows} needs {need}")
    fit = smallest_sufficient_config(n, placed_rows, last_row)
    msg += f"; smallest sufficient config is '{fit.name}'" if fit else "; no built-in config is deep enough"
    raise ConfigError(msg)


# ---- solver.hpp ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Subproblem:
    cur: int = 0
    left: int = 0
    right: int = 0
    placed_rows: int = 0
    multiplier: int = 2


class KernelVariant(enum.Enum):
    iterative = _lib.VARIANT_ITERATIVE
    lastrow = _lib.VARIANT_LASTROW


def to_string(v) -> str:
    return v.name


@dataclass(frozen=True)
class KernelResult:
    count: int = 0
    high_water: int = 0


def pack(subs: Iterable[Subproblem]) -> np.ndarray:
    """Subproblems -> packed 16-byte records (row = placed_rows | multiplier << 8)."""
    subs = list(subs)
    a = np.zeros(len(subs), dtype=SUB_DTYPE)
    for i, s in enumerate(subs):
        a[i] = (s.cur, s.left, s.right, (s.placed_rows & 0xFF) | (s.multiplier << 8))
    return a


def unpack(a: np.ndarray) -> list:
    return [Subproblem(int(r["cols"]), int(r["diag"]), int(r["antidiag"]), int(r["row"]) & 0xFF,
                       int(r["row"]) >> 8) for r in a]


def _check_board(n: int) -> None:
    if n < 1 or n > kMaxBoard:
        raise ConfigError(f"board size must be in [1, 32], got {n}")


# One context per (thread, device) for the single-call helpers below.
_tls = threading.local()


def _ctx(device: int = 0):
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        p = ctypes.c_void_p()
        _call(lib.nq_ctx_create(device, ctypes.byref(p)))
        cache[device] = p
    return cache[device]


def count_each(n: int, subs, variant: KernelVariant = KernelVariant.lastrow, pre_rows: Optional[int] = None,
               device: int = 0):
    """Per-record (count, high_water, nodes) for a batch, on the GPU (nq_count_each)."""
    a = subs if isinstance(subs, np.ndarray) else pack(subs)
    a = np.ascontiguousarray(a, dtype=SUB_DTYPE)
    k = len(a)
    counts = np.zeros(k, dtype=np.uint64)
    high = np.zeros(k, dtype=np.int32)
    nodes = np.zeros(k, dtype=np.uint64)
    if pre_rows is None:
        pre_rows = int((a["row"] & 0xFF).min()) if k else 0
    if k:
        _call(lib.nq_count_each(_ctx(device), n, pre_rows, variant.value, a.ctypes.data, k,
                                counts.ctypes.data, high.ctypes.data, nodes.ctypes.data))
    return counts, high, nodes


def _count_one(variant: KernelVariant, n: int, sub: Subproblem, cfg: StackConfig) -> KernelResult:
    _check_board(n)
    require_feasible(cfg, n, sub.placed_rows, variant is KernelVariant.lastrow)
    c, h, _ = count_each(n, [sub], variant, pre_rows=min(sub.placed_rows, n))
    return KernelResult(int(c[0]), int(h[0]))


def count_iterative(n: int, sub: Subproblem, cfg: StackConfig) -> KernelResult:
    """solver.hpp:79 — Alg. 2 semantics, counted on the GPU."""
    return _count_one(KernelVariant.iterative, n, sub, cfg)


def count_iterative_lastrow(n: int, sub: Subproblem, cfg: StackConfig) -> KernelResult:
    """solver.hpp:138 — Alg. 3 semantics, counted on the GPU."""
    return _count_one(KernelVariant.lastrow, n, sub, cfg)


def count_recursive(n: int, sub: Subproblem) -> int:
    """solver.hpp:69 — the count only (multiplier not applied), counted on the GPU."""
    _check_board(n)
    counts, _, _ = count_each(n, [sub], KernelVariant.iterative, pre_rows=min(sub.placed_rows, n))
    return int(counts[0])


def count_with(variant: KernelVariant, n: int, sub: Subproblem, cfg: StackConfig) -> KernelResult:
    return _count_one(variant, n, sub, cfg)


# ---- subproblems.hpp -----------------------------------------------------------------------
@dataclass
class GenerationPlan:
    n: int = 8
    pre_rows: int = 2
    expected_total: Optional[int] = None


def generate_packed(n: int, pre_rows: int) -> np.ndarray:
    """The folded frontier as packed records, in the reference's stream order."""
    total = ctypes.c_uint64()
    _call(lib.nq_count_subproblems(n, pre_rows, ctypes.byref(total)))
    a = np.zeros(total.value, dtype=SUB_DTYPE)
    got = ctypes.c_uint64()
    _call(lib.nq_generate(n, pre_rows, a.ctypes.data, total.value, ctypes.byref(got)))
    return a


def generate_slice(n: int, pre_rows: int, stride: int, offset: int) -> np.ndarray:
    """Records with stream index ≡ offset (mod stride) — the N=27 projection samples."""
    total = ctypes.c_uint64()
    _call(lib.nq_generate_slice(n, pre_rows, stride, offset, None, 0, ctypes.byref(total)))
    a = np.zeros(total.value, dtype=SUB_DTYPE)
    _call(lib.nq_generate_slice(n, pre_rows, stride, offset, a.ctypes.data, total.value,
                                ctypes.byref(total)))
    return a


def expand(n: int, roots: np.ndarray, target_rows: int) -> np.ndarray:
    """Deepen packed roots to target_rows placed rows (nq_expand): each root's
    descendants in DFS order, roots in order, multiplier inherited."""
    roots = np.ascontiguousarray(roots, dtype=SUB_DTYPE)
    total = ctypes.c_uint64()
    ptr = roots.ctypes.data if len(roots) else None
    _call(lib.nq_expand(n, ptr, len(roots), target_rows, None, 0, ctypes.byref(total)))
    a = np.zeros(total.value, dtype=SUB_DTYPE)
    if total.value:
        _call(lib.nq_expand(n, ptr, len(roots), target_rows, a.ctypes.data, total.value,
                            ctypes.byref(total)))
    return a


def for_each_subproblem(plan: GenerationPlan, sink: Callable[[Subproblem], None]) -> None:
    for s in unpack(generate_packed(plan.n, plan.pre_rows)):
        sink(s)


def generate(plan: GenerationPlan) -> list:
    return unpack(generate_packed(plan.n, plan.pre_rows))


def count_subproblems(n: int, pre_rows: int) -> int:
    total = ctypes.c_uint64()
    _call(lib.nq_count_subproblems(n, pre_rows, ctypes.byref(total)))
    return total.value


def aggregate(results: Sequence) -> int:
    """subproblems.hpp:149-165: Σ multiplier·count, duplicates rejected."""
    seen = set()
    total = 0
    for sub, count in results:
        key = sub.cur
        key = ((key * 0x9E3779B97F4A7C15) & MASK64) ^ sub.left
        key = ((key * 0x9E3779B97F4A7C15) & MASK64) ^ sub.right
        key = ((key * 0x9E3779B97F4A7C15) & MASK64) ^ (sub.placed_rows & MASK64)
        if key in seen:
            raise ConfigError("duplicate subproblem in aggregation input")
        seen.add(key)
        total = checked_add(total, checked_mul(sub.multiplier, count))
    return total


def write_batch(out: io.TextIOBase, plan: GenerationPlan) -> int:
    """subproblems.hpp:169-178: `index cur left right placed_rows multiplier`, hex masks."""
    a = generate_packed(plan.n, plan.pre_rows)
    for i, r in enumerate(a):
        row = int(r["row"])
        out.write(f"{i} {int(r['cols']):x} {int(r['diag']):x} {int(r['antidiag']):x} "
                  f"{row & 0xFF} {row >> 8}\n")
    return len(a)


# ---- scheduler.hpp -------------------------------------------------------------------------
class PartitionStrategy(enum.Enum):
    uniform = _lib.PARTITION_UNIFORM
    weighted = _lib.PARTITION_WEIGHTED
    stealing = _lib.PARTITION_STEALING
    guided = _lib.PARTITION_GUIDED  # GPU extension: shrinking chunks, expensive end first
    strided = _lib.PARTITION_STRIDED  # GPU extension: record i -> worker i mod W, one launch each


def partition_strategy_from(name: str) -> PartitionStrategy:
    try:
        return PartitionStrategy[name]
    except KeyError:
        raise ConfigError(f"unknown partition strategy '{name}'") from None


paper_gpu_weights = (0.20, 0.15, 0.12, 0.11, 0.11, 0.11, 0.10, 0.10)


@dataclass
class PartitionPlan:
    strategy: PartitionStrategy = PartitionStrategy.weighted
    worker_count: int = 1
    weights: list = field(default_factory=list)
    chunk_size: int = 4096


@dataclass(frozen=True)
class IndexRange:
    first: int = 0
    last: int = 0

    def size(self) -> int:
        return self.last - self.first


def _ranges(buf, k):
    return [IndexRange(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(k)]


def partition_uniform(task_count: int, worker_count: int) -> list:
    if worker_count < 1:
        raise ConfigError("worker_count must be >= 1")
    buf = (ctypes.c_uint64 * (2 * worker_count))()
    _call(lib.nq_partition_uniform(task_count, worker_count, buf))
    return _ranges(buf, worker_count)


def partition_weighted(task_count: int, weights: Sequence[float]) -> list:
    if not weights:
        raise ConfigError("weighted partition needs at least one weight")
    w = (ctypes.c_double * len(weights))(*weights)
    buf = (ctypes.c_uint64 * (2 * len(weights)))()
    _call(lib.nq_partition_weighted(task_count, w, len(weights), buf))
    return _ranges(buf, len(weights))


@dataclass
class WorkerStats:
    worker: int = 0
    assigned: int = 0
    processed: int = 0
    partial_sum: int = 0
    elapsed_ms: float = 0.0
    device: int = 0
    nodes: int = 0
    kernel_ms: float = 0.0
    chunks: int = 0
    span_ms: float = 0.0  # device time, first enqueued operation -> last kernel end
    launches: int = 0     # kernel launches (dynamic strategies: one streaming launch)


@dataclass
class SolveReport:
    n: int = 0
    pre_rows: int = 0
    config_name: str = ""
    kernel: KernelVariant = KernelVariant.lastrow
    strategy: PartitionStrategy = PartitionStrategy.weighted
    worker_count: int = 1
    task_count: int = 0
    generation_ms: float = 0.0
    calc_ms: float = 0.0
    total: int = 0
    completed: bool = True
    workers: list = field(default_factory=list)
    nodes: int = 0

    def skew_ratio(self) -> float:
        lo = hi = 0.0
        for w in self.workers:
            hi = max(hi, w.elapsed_ms)
            if lo == 0 or (0 < w.elapsed_ms < lo):
                lo = w.elapsed_ms
        return hi / lo if lo > 0 else 0.0

    def to_json(self) -> dict:
        return {"n": self.n, "pre_rows": self.pre_rows, "config": self.config_name,
                "kernel": self.kernel.name, "partition": self.strategy.name,
                "worker_count": self.worker_count, "task_count": self.task_count,
                "generation_ms": self.generation_ms, "calc_ms": self.calc_ms,
                "total": self.total, "completed": self.completed,
                "skew_ratio": self.skew_ratio(), "nodes": self.nodes,
                "workers": [{"worker": w.worker, "assigned": w.assigned, "processed": w.processed,
                             "partial_sum": w.partial_sum, "elapsed_ms": w.elapsed_ms,
                             "device": w.device, "nodes": w.nodes} for w in self.workers]}


def _log_line(kind: int, i: int, u: int, d: float) -> str:
    buf = ctypes.create_string_buffer(256)
    _call(lib.nq_format_log(kind, i, u, d, buf, 256))
    return buf.value.decode()


def log_generation_line(ms: float, count: int) -> str:
    return _log_line(_lib.LOG_GENERATION, 0, count, ms)


def log_start_line(worker: int, count: int, fraction: float) -> str:
    return _log_line(_lib.LOG_START, worker, count, fraction)


def log_finish_line(worker: int) -> str:
    return _log_line(_lib.LOG_FINISH, worker, 0, 0.0)


def log_result_line(n: int, total: int, calc_ms: float) -> str:
    return _log_line(_lib.LOG_RESULT, n, total, calc_ms)


@dataclass
class ExecuteOptions:
    kernel: KernelVariant = KernelVariant.lastrow
    config: StackConfig = builtin_configs[1]  # config2 (scheduler.hpp:248)
    plan: PartitionPlan = field(default_factory=PartitionPlan)
    log: Optional[Callable[[str], None]] = None
    progress: object = None
    cancel: Optional[threading.Event] = None
    resume: list = field(default_factory=list)
    devices: Optional[Sequence[int]] = None  # GPU extension: explicit device list
    dispatch: Optional["Dispatcher"] = None  # GPU extension: shared dynamic dispenser


class _CancelWatch:
    """Copies a threading.Event into the int the C scheduler polls between chunks
    (the ExecuteOptions::cancel atomic of scheduler.hpp:252), until stopped."""

    def __init__(self, event: threading.Event, flag: ctypes.c_int):
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                if event.wait(0.001):
                    flag.value = 1
                    return
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        self._t.join()


def _stop_watchers(keep: list) -> None:
    for k in keep:
        if isinstance(k, _CancelWatch):
            k.stop()


def _solve_opts(opts: ExecuteOptions, keep: list):
    if opts.progress is not None or opts.resume:
        raise ConfigError("checkpoint progress/resume is not supported on the GPU path yet")
    o = _lib.NqSolveOpts()
    o.variant = opts.kernel.value
    o.strategy = opts.plan.strategy.value
    o.worker_count = opts.plan.worker_count
    if opts.plan.strategy is PartitionStrategy.weighted and opts.plan.weights:
        if len(opts.plan.weights) != opts.plan.worker_count:
            raise ConfigError("weights length must equal worker_count")
        w = (ctypes.c_double * len(opts.plan.weights))(*opts.plan.weights)
        keep.append(w)
        o.weights = w
    o.chunk = opts.plan.chunk_size
    if opts.devices:
        d = (ctypes.c_int * len(opts.devices))(*opts.devices)
        keep.append(d)
        o.devices = d
        o.n_devices = len(opts.devices)
    if opts.dispatch is not None:
        o.dispatch = opts.dispatch.handle
    o.stack_depth = opts.config.max_depth()
    name = opts.config.name.encode()
    keep.append(name)
    o.config_name = name
    if opts.cancel is not None:
        flag = ctypes.c_int(1 if opts.cancel.is_set() else 0)
        keep.append(flag)
        o.cancel = ctypes.pointer(flag)
        keep.append(o.cancel)
        keep.append(_CancelWatch(opts.cancel, flag))
    if opts.log is not None:
        sink = opts.log
        cb = _lib.NQ_LOG_FN(lambda _u, line: sink(line.decode()))
        keep.append(cb)
        o.log = cb
    return o


def _report(n: int, pre_rows: int, opts: ExecuteOptions, rep) -> SolveReport:
    r = SolveReport(n=n, pre_rows=pre_rows, config_name=opts.config.name, kernel=opts.kernel,
                    strategy=opts.plan.strategy, worker_count=rep.worker_count,
                    task_count=rep.task_count, generation_ms=rep.generation_ms,
                    calc_ms=rep.calc_ms, total=rep.total, completed=bool(rep.completed),
                    nodes=rep.nodes)
    for i in range(rep.worker_count):
        w = rep.workers[i]
        r.workers.append(WorkerStats(worker=w.worker, assigned=w.assigned, processed=w.processed,
                                     partial_sum=w.partial_sum, elapsed_ms=w.elapsed_ms,
                                     device=w.device, nodes=w.nodes, kernel_ms=w.kernel_ms,
                                     chunks=w.chunks, span_ms=w.span_ms, launches=w.launches))
    return r


def execute_batch(n: int, pre_rows: int, batch, opts: ExecuteOptions) -> SolveReport:
    """scheduler.hpp:266 on the GPUs: every record exactly once, totals strategy-invariant."""
    if opts.plan.worker_count < 1:
        raise ConfigError("worker_count must be >= 1")
    if opts.plan.strategy is PartitionStrategy.stealing and opts.plan.chunk_size == 0:
        raise ConfigError("chunk_size must be >= 1")
    require_feasible(opts.config, n, pre_rows, opts.kernel is KernelVariant.lastrow)
    a = batch if isinstance(batch, np.ndarray) else pack(batch)
    a = np.ascontiguousarray(a, dtype=SUB_DTYPE)
    keep: list = []
    o = _solve_opts(opts, keep)
    rep = _lib.NqReport()
    try:
        _call(lib.nq_solve_batch(n, pre_rows, a.ctypes.data if len(a) else None, len(a),
                                 ctypes.byref(o), ctypes.byref(rep)))
    finally:
        _stop_watchers(keep)
    return _report(n, pre_rows, opts, rep)


def execute_batch_device(n: int, pre_rows: int, dev_ptrs: Sequence[int], count: int,
                         opts: ExecuteOptions) -> SolveReport:
    """execute_batch over a frontier already resident on every worker device
    (nq_solve_batch_device): dev_ptrs[i] holds all `count` packed records on the i-th
    device of opts.devices; workers launch on sub-ranges, only results cross PCIe."""
    if opts.plan.worker_count < 1:
        raise ConfigError("worker_count must be >= 1")
    require_feasible(opts.config, n, pre_rows, opts.kernel is KernelVariant.lastrow)
    keep: list = []
    o = _solve_opts(opts, keep)
    ptrs = (ctypes.c_void_p * len(dev_ptrs))(*dev_ptrs)
    rep = _lib.NqReport()
    try:
        _call(lib.nq_solve_batch_device(n, pre_rows, ptrs, count, ctypes.byref(o), ctypes.byref(rep)))
    finally:
        _stop_watchers(keep)
    return _report(n, pre_rows, opts, rep)


def execute_batch_expand(n: int, target_rows: int, roots, opts: ExecuteOptions) -> SolveReport:
    """execute_batch over roots that every worker deepens to target_rows on its own
    device first (nq_solve_batch_expand; strided or guided): only the roots cross PCIe.
    Same totals and Alg. 3 nodes as counting the deepened records."""
    if opts.plan.worker_count < 1:
        raise ConfigError("worker_count must be >= 1")
    require_feasible(opts.config, n, target_rows, opts.kernel is KernelVariant.lastrow)
    a = roots if isinstance(roots, np.ndarray) else pack(roots)
    a = np.ascontiguousarray(a, dtype=SUB_DTYPE)
    keep: list = []
    o = _solve_opts(opts, keep)
    rep = _lib.NqReport()
    try:
        _call(lib.nq_solve_batch_expand(n, target_rows, a.ctypes.data if len(a) else None, len(a),
                                        ctypes.byref(o), ctypes.byref(rep)))
    finally:
        _stop_watchers(keep)
    r = _report(n, target_rows, opts, rep)
    return r


class Dispatcher:
    """The scheduler's host-side dynamic chunk dispenser (nq_dispatch_*). name=None: private
    to this process; a name: a POSIX shared-memory segment that cooperating processes
    (one per GPU) attach to, so they share ONE guided/stealing cursor with no device
    collective (scheduler.hpp:351-362). Partials are posted per slot and summed checked."""

    def __init__(self, handle: int, name: Optional[str], owner: bool):
        self.handle = handle
        self.name = name
        self._owner = owner

    @classmethod
    def create(cls, count: int, strategy: PartitionStrategy = PartitionStrategy.guided,
               chunk: int = 0, workers: int = 1, name: Optional[str] = None) -> "Dispatcher":
        h = ctypes.c_void_p()
        _call(lib.nq_dispatch_create(name.encode() if name else None, count, strategy.value,
                                     chunk, workers, ctypes.byref(h)))
        return cls(h.value, name, True)

    @classmethod
    def attach(cls, name: str) -> "Dispatcher":
        h = ctypes.c_void_p()
        _call(lib.nq_dispatch_attach(name.encode(), ctypes.byref(h)))
        return cls(h.value, name, False)

    def take(self):
        """(first, length) of the next chunk, or None when drained."""
        f, n = ctypes.c_uint64(), ctypes.c_uint64()
        rc = lib.nq_dispatch_take(self.handle, ctypes.byref(f), ctypes.byref(n))
        if rc < 0:
            _call(rc)
        return (f.value, n.value) if rc == 1 else None

    def reset(self) -> None:
        _call(lib.nq_dispatch_reset(self.handle))

    def info(self) -> dict:
        c, s, k, w = ctypes.c_uint64(), ctypes.c_int(), ctypes.c_uint64(), ctypes.c_int()
        _call(lib.nq_dispatch_info(self.handle, ctypes.byref(c), ctypes.byref(s), ctypes.byref(k),
                                   ctypes.byref(w)))
        return {"count": c.value, "strategy": PartitionStrategy(s.value), "chunk": k.value,
                "workers": w.value}

    def post(self, slot: int, solutions: int, nodes: int, processed: int) -> None:
        _call(lib.nq_dispatch_post(self.handle, slot, solutions, nodes, processed))

    def sum(self, slots: int):
        """(solutions, nodes, processed) over slots 0..slots-1 (every slot must have posted)."""
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _call(lib.nq_dispatch_sum(self.handle, slots, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def close(self, unlink: Optional[bool] = None) -> None:
        if self.handle:
            lib.nq_dispatch_close(self.handle, int(self._owner if unlink is None else unlink))
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def execute(n: int, pre_rows: int, opts: ExecuteOptions) -> SolveReport:
    """scheduler.hpp:393: generate + execute_batch (n == 1 short-circuits to Q(1) = 1)."""
    _check_board(n)
    if n > 1:
        require_feasible(opts.config, n, pre_rows, opts.kernel is KernelVariant.lastrow)
    keep: list = []
    o = _solve_opts(opts, keep)
    rep = _lib.NqReport()
    try:
        _call(lib.nq_solve(n, pre_rows, ctypes.byref(o), ctypes.byref(rep)))
    finally:
        _stop_watchers(keep)
    r = _report(n, 0 if n == 1 else pre_rows, opts, rep)
    if n == 1:
        r.workers = [WorkerStats(worker=w) for w in range(opts.plan.worker_count)]
        r.workers[0].partial_sum = 1
        r.worker_count = opts.plan.worker_count
    return r


def execute_checkpointed(n: int, pre_rows: int, opts: ExecuteOptions, path: str, chunk: int = 0,
                         flush_interval_s: float = 0.0, resume: bool = False,
                         stop_after_s: float = 0.0) -> SolveReport:
    """execute() with chunk-granular checkpoint/resume (nq_solve_checkpointed; the GPU
    counterpart of run_with_checkpoint, runner.hpp:48-212). Workers take pending chunks;
    a cancel leaves completed = False and a file a later resume=True call continues."""
    _check_board(n)
    require_feasible(opts.config, n, pre_rows, opts.kernel is KernelVariant.lastrow)
    plan = opts.plan
    o_opts = ExecuteOptions(kernel=opts.kernel, config=opts.config,
                            plan=PartitionPlan(PartitionStrategy.stealing, plan.worker_count, [], 1),
                            log=opts.log, cancel=opts.cancel, devices=opts.devices)
    keep: list = []
    o = _solve_opts(o_opts, keep)
    ck = _lib.NqCkptOpts(str(path).encode(), chunk, flush_interval_s, 1 if resume else 0,
                         stop_after_s)
    rep = _lib.NqReport()
    try:
        _call(lib.nq_solve_checkpointed(n, pre_rows, ctypes.byref(o), ctypes.byref(ck), ctypes.byref(rep)))
    finally:
        _stop_watchers(keep)
    r = _report(n, pre_rows, o_opts, rep)
    r.strategy = plan.strategy
    return r


@dataclass
class RunSpec:
    """runner.hpp:20-26."""
    n: int = 8
    pre_rows: int = 2
    config: StackConfig = builtin_configs[1]
    kernel: KernelVariant = KernelVariant.lastrow
    plan: PartitionPlan = field(default_factory=PartitionPlan)


@dataclass
class CheckpointOptions:
    """runner.hpp:28-32; flush_interval = records per recorded chunk on the GPU path."""
    path: str = ""
    flush_interval: int = 1_000_000
    resume: bool = False


def run_with_checkpoint(spec: RunSpec, ckpt: CheckpointOptions, cancel=None, log=None) -> SolveReport:
    """runner.hpp:48-212 over the chunk-granular GPU checkpoint (execute_checkpointed),
    with the reference's validation (stealing refused, n == 1 short-circuit)."""
    if spec.plan.strategy is PartitionStrategy.stealing:
        raise ConfigError("checkpointing requires a contiguous partition (uniform/weighted)")
    _check_board(spec.n)
    opts = ExecuteOptions(kernel=spec.kernel, config=spec.config, plan=spec.plan, log=log,
                          cancel=cancel)
    if spec.n == 1:
        return execute(1, 0, opts)
    if ckpt.flush_interval < 1:
        raise ConfigError("flush_interval must be >= 1")
    r = execute_checkpointed(spec.n, spec.pre_rows, opts, ckpt.path, chunk=ckpt.flush_interval,
                             resume=ckpt.resume)
    if r.completed and log is not None:
        log(log_result_line(spec.n, r.total, r.calc_ms))
    return r


def checkpoint_info(path: str):
    """(n, pre_rows, chunks, done_chunks) recorded in a checkpoint file."""
    d = checkpoint_details(path)
    return d["n"], d["pre_rows"], d["chunks"], d["done_chunks"]


def checkpoint_details(path: str) -> dict:
    """Every run parameter a checkpoint records (n, pre_rows, kernel, chunk) and its
    progress; a resume must repeat n, R, kernel and chunk (the file's identity)."""
    n, r, v = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    chunk, chunks, done = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _call(lib.nq_checkpoint_info(str(path).encode(), ctypes.byref(n), ctypes.byref(r), ctypes.byref(v),
                                 ctypes.byref(chunk), ctypes.byref(chunks), ctypes.byref(done)))
    return {"n": n.value, "pre_rows": r.value, "kernel": KernelVariant(v.value), "chunk": chunk.value,
            "chunks": chunks.value, "done_chunks": done.value}


def measure_int_peak(device: int = 0):
    """(thread int-ops/s, SM MHz) of a LOP3+IMAD 1:1 stream on all SMs."""
    ops = ctypes.c_double()
    mhz = ctypes.c_double()
    _call(lib.nq_measure_int_peak(device, ctypes.byref(ops), ctypes.byref(mhz)))
    return ops.value, mhz.value


def device_count() -> int:
    n = ctypes.c_int()
    _call(lib.nq_device_count(ctypes.byref(n)))
    return n.value

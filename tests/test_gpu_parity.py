"""GPU parity: the sm_100a DFS kernel through the C ABI vs the reference (golden
vectors recorded from the reference build), the C oracle, OEIS A000170 and the
Appendix-B node counts. Bit-exact throughout (integer path).

Mirrors test_solver.cpp, test_scheduler.cpp and acceptance.cpp criteria 1, 3, 4, 7, 9.
"""
import ctypes
import threading

import numpy as np
import pytest

from paper_2511_12009_b200 import _lib
from paper_2511_12009_b200 import nqueens as nq

pytestmark = pytest.mark.gpu

CFG1 = nq.builtin_configs[0]


def as_recs(lst):
    return np.array([tuple(r) for r in lst], dtype=_lib.SUB_DTYPE)


class Ctx:
    def __init__(self, block=0, bps=0, reverse=1, layout=_lib.LAYOUT_V4, balance=1):
        self.p = ctypes.c_void_p()
        _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(self.p)))
        _lib.check(_lib.lib.nq_ctx_set_layout(self.p, layout))
        _lib.check(_lib.lib.nq_ctx_set_balance(self.p, balance))
        _lib.check(_lib.lib.nq_ctx_set_tuning(self.p, block, bps, reverse))

    def count(self, n, pre_rows, a, variant=_lib.VARIANT_LASTROW):
        r = _lib.NqResult()
        _lib.check(_lib.lib.nq_count(self.p, n, pre_rows, variant, a.ctypes.data if len(a) else None,
                                     len(a), ctypes.byref(r)))
        return r

    def close(self):
        _lib.lib.nq_ctx_destroy(self.p)


def test_per_subproblem_vs_reference_golden(golden):
    """Every subproblem n<=12, R in {1,2,3}: count + high_water, iterative and lastrow
    (test_solver.cpp:70-80, :92-103, :116-134; acceptance criterion 3)."""
    for key, d in golden["per_subproblem"].items():
        n, r = map(int, key.split(","))
        a = as_recs(d["records"])
        for variant, ref in (("iterative", d["iterative"]), ("lastrow", d["lastrow"])):
            c, h, _ = nq.count_each(n, a, nq.KernelVariant[variant], pre_rows=r)
            assert c.tolist() == [x[0] for x in ref], (key, variant)
            assert h.tolist() == [x[1] for x in ref], (key, variant)
        c, _, _ = nq.count_each(n, a, nq.KernelVariant.iterative, pre_rows=r)
        assert c.tolist() == d["recursive"]


def test_per_subproblem_nodes_vs_oracle(oracle):
    """Alg. 3 node counts per subproblem equal the oracle's loop iterations."""
    for n, r in [(10, 3), (12, 4), (14, 5)]:
        a = oracle.generate(n, r)
        c, h, nodes = nq.count_each(n, a, nq.KernelVariant.lastrow, pre_rows=r)
        for i in range(0, len(a), max(1, len(a) // 300)):
            oc, oh, on = oracle.count_lastrow(n, tuple(int(x) for x in a[i]))
            assert (int(c[i]), int(h[i]), int(nodes[i])) == (oc, oh, on), (n, r, i)


def test_shallow_roots_and_full_boards():
    # test_solver.cpp:82-90, :105-114
    sol = [0, 2, 4, 1, 3]
    cur = left = right = 0
    for col in sol:
        s = nq.apply_placement(cur, left, right, 1 << col)
        cur, left, right = s.cur, s.left, s.right
    sub = nq.Subproblem(cur, left, right, 5, 1)
    assert cur == nq.board_mask(5)
    assert nq.count_iterative(5, sub, CFG1).count == 1
    assert nq.count_iterative_lastrow(5, sub, CFG1).count == 1
    assert nq.count_iterative_lastrow(1, nq.Subproblem(), CFG1).count == 1
    assert nq.count_iterative_lastrow(4, nq.Subproblem(), CFG1).count == 2
    for n in (1, 2, 3):
        assert nq.count_recursive(n, nq.Subproblem()) == [1, 0, 0][n - 1]


def test_q_of_n_1_to_18(golden):
    """acceptance criterion 1 / 9 at GPU sizes."""
    for n in range(1, 19):
        r = min(6, n - 1) if n > 1 else 1
        rep = nq.execute(n, r, nq.ExecuteOptions(config=CFG1))
        assert rep.total == golden["oeis_a000170"][n - 1], n
        assert rep.completed


def test_node_counts_appendix_b(golden):
    """Device node counter == Appendix B (exact, reference generator) for N=14..20,
    R=5..7 (the N=20 profile took 47 min on 8 cores to derive)."""
    for n in range(14, 21):
        for r, nodes in golden["appendix_b_nodes"][str(n)].items():
            rep = nq.execute(n, int(r), nq.ExecuteOptions(config=CFG1))
            assert rep.total == golden["oeis_a000170"][n - 1]
            assert rep.nodes == nodes, (n, r)


def test_q21_bit_exact(golden):
    """Q(21) = 314 666 222 712 through execute() (~13 s on one B200), pinned to OEIS
    A000170. The node counter at this N is pinned independently on the slice
    i ≡ 0 (mod 1000) of the same frontier, against the C oracle on the records the
    reference's own generator picks (test_bench_samples_rederived_on_device); the
    full-count node total must agree with the slice's per-record density to 1%."""
    import json
    import os
    rep = nq.execute(21, 7, nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.strided, 1)))
    assert rep.total == golden["oeis_a000170"][20] == 314666222712
    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_samples.json")) as f:
        sl = json.load(f)["21,7,1000"]
    assert abs(rep.nodes / (sl["nodes"] * 1000) - 1) < 0.01


@pytest.mark.slow
def test_q22_through_execute_device_deepening(golden):
    """BASELINE configs[3]: Q(22) = 2 691 008 701 644 through execute() on one B200
    (~118 s): the coarse R=4 frontier is dealt out and deepened to R=7 on the device."""
    rep = nq.execute(22, 7, nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.strided, 1)))
    assert rep.total == golden["oeis_a000170"][21] == 2691008701644
    assert rep.completed and rep.task_count == 60760010


@pytest.mark.slow
def test_n20_full(golden):
    rep = nq.execute(20, 6, nq.ExecuteOptions(config=CFG1))
    assert rep.total == 39029188884
    assert rep.nodes == golden["appendix_b_nodes"]["20"]["6"]


def test_totals_invariant_across_strategies_and_workers():
    """test_scheduler.cpp:77-111: exactly-once processing, partial sums add up."""
    expected = nq.execute(12, 2, nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.uniform, 1))).total
    assert expected == 14200
    for strategy in nq.PartitionStrategy:
        for workers in (1, 2, 4, 8):
            plan = nq.PartitionPlan(strategy, workers, [], 3)
            if strategy is nq.PartitionStrategy.weighted and workers == 8:
                plan.weights = list(nq.paper_gpu_weights)
            rep = nq.execute(12, 2, nq.ExecuteOptions(plan=plan))
            assert rep.total == expected and rep.completed
            assert sum(w.processed for w in rep.workers) == rep.task_count
            assert sum(w.partial_sum for w in rep.workers) == rep.total
            if strategy in (nq.PartitionStrategy.uniform, nq.PartitionStrategy.weighted):
                assert sum(w.assigned for w in rep.workers) == rep.task_count
            if strategy in (nq.PartitionStrategy.stealing, nq.PartitionStrategy.guided):
                assert all(w.assigned == 0 for w in rep.workers)  # 0 = dynamic (:106)


def test_kernel_flag_same_totals():
    # test_scheduler.cpp:113-119
    a = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.uniform, 2))
    b = nq.ExecuteOptions(kernel=nq.KernelVariant.iterative,
                          plan=nq.PartitionPlan(nq.PartitionStrategy.uniform, 2))
    assert nq.execute(11, 3, a).total == nq.execute(11, 3, b).total == 2680


def test_n1_short_circuit():
    rep = nq.execute(1, 1, nq.ExecuteOptions())
    assert rep.total == 1 and rep.workers[0].partial_sum == 1


def test_log_lines_emitted():
    lines = []
    rep = nq.execute(10, 3, nq.ExecuteOptions(log=lines.append,
                                              plan=nq.PartitionPlan(nq.PartitionStrategy.stealing, 2, [], 16)))
    assert rep.total == 724
    assert any("generate" in l for l in lines)
    assert sum("start job" in l for l in lines) == 2 and sum("finish job" in l for l in lines) == 2
    assert "n 10 queens result 724, calc time:" in lines[-1]


def test_cancel_before_start():
    ev = threading.Event()
    ev.set()
    rep = nq.execute(12, 3, nq.ExecuteOptions(cancel=ev, plan=nq.PartitionPlan(nq.PartitionStrategy.stealing, 2, [], 8)))
    assert not rep.completed


def test_tuning_variants_identical(oracle):
    a = oracle.generate(15, 5)
    base = None
    for layout, balance in ((_lib.LAYOUT_V4, 1), (_lib.LAYOUT_V4, 0), (_lib.LAYOUT_PLANES, 1)):
        for block in (64, 96, 128, 192, 256):
            for reverse in (0, 1):
                for bps in (0, 1):
                    c = Ctx(block, bps, reverse, layout, balance)
                    r = c.count(15, 5, a)
                    c.close()
                    got = (r.solutions, r.raw_solutions, r.nodes, r.subproblems)
                    base = base or got
                    assert got == base, (layout, balance, block, reverse, bps)
    assert base[0] == 2279184 and base[3] == len(a)


def test_planes_layout_per_subproblem(oracle):
    """The zero-bank-conflict plane layout gives the same per-record results."""
    a = oracle.generate(12, 3)
    want = nq.count_each(12, a, nq.KernelVariant.lastrow, pre_rows=3)
    c = Ctx(layout=_lib.LAYOUT_PLANES)
    r = c.count(12, 3, a)
    c.close()
    assert r.solutions == 14200 and r.nodes == int(want[2].sum())


def test_random_subsets_and_permutations(oracle):
    """Order and batch composition never change a per-record result."""
    rng = np.random.default_rng(2511)
    a = oracle.generate(14, 4)
    ref_counts = oracle.solve_batch(14, a, per_sub=True)[2]
    for _ in range(4):
        idx = rng.permutation(len(a))[: rng.integers(1, len(a))]
        c, _, _ = nq.count_each(14, a[idx], nq.KernelVariant.lastrow, pre_rows=4)
        assert np.array_equal(c, ref_counts[idx])


def test_mixed_depth_batch(oracle):
    """Records of different placed_rows in one launch (stack sized by the minimum)."""
    parts = [oracle.generate(13, r) for r in (2, 3, 4)]
    a = np.concatenate(parts)
    ctx = Ctx()
    r = ctx.count(13, 2, a)
    ctx.close()
    assert r.solutions == 3 * 73712


def test_empty_and_rejected_batches():
    ctx = Ctx()
    r = ctx.count(10, 3, np.zeros(0, dtype=_lib.SUB_DTYPE))
    assert r.solutions == 0 and r.subproblems == 0
    bad = nq.generate_packed(10, 3)
    bad[5]["cols"] |= 1 << 12  # outside the board
    with pytest.raises(_lib.NqError) as e:
        ctx.count(10, 3, bad)
    assert e.value.code == _lib.NQ_ECONFIG and "record 5" in str(e.value)
    shallow = nq.generate_packed(10, 2)
    with pytest.raises(_lib.NqError):
        ctx.count(10, 3, shallow)  # placed_rows below the declared pre_rows
    ctx.close()
    for strategy in (nq.PartitionStrategy.uniform, nq.PartitionStrategy.strided,
                     nq.PartitionStrategy.guided, nq.PartitionStrategy.stealing):
        opts = nq.ExecuteOptions(plan=nq.PartitionPlan(strategy, 2, [], 16))
        with pytest.raises(RuntimeError) as e:
            nq.execute_batch(10, 3, bad, opts)
        # streaming launches report the queue position; the scheduler maps it back
        assert "failed on subproblem 5" in str(e.value), (strategy, str(e.value))


def test_pinned_host_batch_is_read_in_place(golden):
    """A page-locked host batch is read by the kernel over the bus (no H2D copy); a
    pageable one is copied. Same counts either way, through nq_count and through the
    scheduler (two workers on device 0: streaming launches publishing host chunks), and
    a malformed record in pinned memory is still rejected by index."""
    import torch
    n, r = 18, 6
    recs = nq.generate_packed(n, r)
    pinned = torch.from_numpy(recs.view(np.int32).reshape(-1, 4).copy()).pin_memory()
    ctx = Ctx()
    a = ctx.count(n, r, recs)                                  # pageable: copied
    b = _lib.NqResult()
    _lib.check(_lib.lib.nq_count(ctx.p, n, r, _lib.VARIANT_LASTROW,
                                 ctypes.c_void_p(pinned.data_ptr()), len(recs), ctypes.byref(b)))
    assert (a.solutions, a.nodes) == (b.solutions, b.nodes) == (golden["oeis_a000170"][n - 1], golden["appendix_b_nodes"][str(n)][str(r)])
    assert a.h2d_ms > 1.0 and b.h2d_ms < 0.5, (a.h2d_ms, b.h2d_ms)
    o = _lib.NqSolveOpts()
    o.variant = _lib.VARIANT_LASTROW
    o.strategy = _lib.PARTITION_GUIDED
    o.worker_count = 2
    devs = (ctypes.c_int * 2)(0, 0)
    o.devices = devs
    o.n_devices = 2
    rep = _lib.NqReport()
    _lib.check(_lib.lib.nq_solve_batch(n, r, ctypes.c_void_p(pinned.data_ptr()), len(recs),
                                       ctypes.byref(o), ctypes.byref(rep)))
    assert (rep.total, rep.nodes) == (golden["oeis_a000170"][n - 1], golden["appendix_b_nodes"][str(n)][str(r)])
    bad = pinned.clone().pin_memory()
    bad[7, 0] = int(np.int32(-1))                              # cols outside the board
    with pytest.raises(_lib.NqError) as e:
        _lib.check(_lib.lib.nq_count(ctx.p, n, r, _lib.VARIANT_LASTROW,
                                     ctypes.c_void_p(bad.data_ptr()), len(recs), ctypes.byref(b)))
    assert "record 7" in str(e.value)
    ctx.close()


def test_device_resident_async_path(oracle):
    import torch
    a = oracle.generate(16, 5)
    d = torch.from_numpy(a.view(np.uint32).reshape(-1, 4).astype(np.int32)).cuda()
    ctx = Ctx()
    _lib.check(_lib.lib.nq_count_device_async(ctx.p, 16, 5, 1, ctypes.c_void_p(d.data_ptr()), len(a)))
    r = _lib.NqResult()
    _lib.check(_lib.lib.nq_collect(ctx.p, ctypes.byref(r)))
    assert r.solutions == 14772512
    r2 = _lib.NqResult()
    _lib.check(_lib.lib.nq_count_device(ctx.p, 16, 5, 1, ctypes.c_void_p(d.data_ptr()), len(a),
                                        ctypes.byref(r2)))
    assert (r2.solutions, r2.nodes) == (r.solutions, r.nodes) == (14772512, 563126914)
    ctx.close()


def test_int_peak_measurement():
    ops, mhz = nq.measure_int_peak(0)
    assert 5e12 < ops < 1e14 and 500 < mhz < 2500


def test_cancel_mid_run_stops_between_chunks():
    """A cancel raised while the GPUs are counting stops dispatch at the next chunk
    boundary (scheduler.hpp:342-355); the report says completed = False."""
    import threading
    import time
    ev = threading.Event()
    opts = nq.ExecuteOptions(cancel=ev, plan=nq.PartitionPlan(nq.PartitionStrategy.stealing, 2, [], 2048))
    timer = threading.Timer(0.05, ev.set)
    timer.start()
    t0 = time.perf_counter()
    rep = nq.execute(19, 6, opts)
    timer.cancel()
    assert not rep.completed
    assert sum(w.processed for w in rep.workers) < rep.task_count
    assert time.perf_counter() - t0 < 30


def test_cancel_during_a_streaming_launch():
    """Guided dispatch feeds ONE streaming launch; a cancel makes the feeder stop
    publishing and close the queue: what was already published (at most about one guided
    chunk) is counted, the rest is not, and the report says completed = False."""
    import threading
    import time
    batch = nq.generate_packed(21, 7)                     # ~13 s of work on one B200
    ev = threading.Event()
    # two workers (both on device 0): one worker alone gets the contiguous launch
    opts = nq.ExecuteOptions(cancel=ev, plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 2),
                             devices=[0, 0])
    assert nq.execute(12, 4, nq.ExecuteOptions(plan=opts.plan, devices=[0, 0])).total == 14200
    timer = threading.Timer(1.0, ev.set)
    timer.start()
    t0 = time.perf_counter()
    rep = nq.execute_batch(21, 7, batch, opts)
    dt = time.perf_counter() - t0
    timer.cancel()
    assert not rep.completed
    assert all(w.launches == 1 for w in rep.workers)
    assert 0 < sum(w.processed for w in rep.workers) < len(batch)
    assert dt < 6.5, dt


def test_cancel_inside_a_running_launch():
    """With the strided strategy each worker is ONE persistent launch; a cancel raised
    while it runs reaches the kernel through the device stop word (nq_ctx_set_cancel):
    dispatch stops at the next refill, lanes finish the subtree they hold."""
    import threading
    import time
    opts0 = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.strided, 1))
    assert nq.execute(12, 4, opts0).total == 14200        # context, module, pool warm
    batch = nq.generate_packed(21, 7)                     # ~13 s of work on one B200
    ev = threading.Event()
    opts = nq.ExecuteOptions(cancel=ev, plan=nq.PartitionPlan(nq.PartitionStrategy.strided, 1))
    timer = threading.Timer(1.0, ev.set)
    timer.start()
    t0 = time.perf_counter()
    rep = nq.execute_batch(21, 7, batch, opts)
    dt = time.perf_counter() - t0
    timer.cancel()
    assert not rep.completed
    assert 0 < rep.workers[0].processed < len(batch)
    assert dt < 4.0, dt


def test_device_expansion_matches_host_expand():
    """GPU-side frontier deepening (nq_expand_device) writes exactly the host nq_expand
    stream, and nq_count_expand (coarse roots -> device deepening -> DFS) counts Q(n)."""
    import torch
    for n, r0, r1 in ((9, 2, 5), (13, 2, 6), (16, 4, 7), (18, 3, 7)):
        roots = nq.generate_packed(n, r0)
        want = nq.expand(n, roots, r1)
        d_roots = torch.from_numpy(roots.view(np.int32).reshape(-1, 4)).cuda()
        total = ctypes.c_uint64()
        _lib.check(_lib.lib.nq_expand_device(0, n, ctypes.c_void_p(d_roots.data_ptr()), len(roots), r1,
                                             None, 0, ctypes.byref(total)))
        assert total.value == len(want)
        d_out = torch.zeros((len(want), 4), dtype=torch.int32, device="cuda")
        _lib.check(_lib.lib.nq_expand_device(0, n, ctypes.c_void_p(d_roots.data_ptr()), len(roots), r1,
                                             ctypes.c_void_p(d_out.data_ptr()), len(want),
                                             ctypes.byref(total)))
        got = d_out.cpu().numpy().view(_lib.SUB_DTYPE).reshape(-1)
        assert np.array_equal(got, want), (n, r0, r1)
    c = Ctx()
    r = _lib.NqResult()
    roots = nq.generate_packed(18, 4)
    _lib.check(_lib.lib.nq_count_expand(c.p, 18, 7, _lib.VARIANT_LASTROW, roots.ctypes.data, len(roots),
                                        ctypes.byref(r)))
    assert r.solutions == 666090624 and r.subproblems == nq.count_subproblems(18, 7)
    assert r.nodes == 29341087800  # Appendix B, R=7
    bad = roots.copy()
    bad["row"][3] += 1
    with pytest.raises(_lib.NqError) as e:
        _lib.check(_lib.lib.nq_count_expand(c.p, 18, 7, _lib.VARIANT_LASTROW, bad.ctypes.data, len(bad),
                                            ctypes.byref(r)))
    assert "root 3" in str(e.value)
    c.close()


def _random_deep_records(n, depth, k, rng):
    """k random valid partial placements with `depth` queens (random descent, restarts
    on dead ends), packed like the generator's records (multiplier 2)."""
    mask = (1 << n) - 1
    out = []
    while len(out) < k:
        cur = left = right = 0
        for _ in range(depth):
            v = mask & ~(cur | left | right)
            if not v:
                break
            bits = [b for b in range(n) if v >> b & 1]
            p = 1 << int(rng.choice(bits))
            cur, left, right = cur | p, ((left | p) << 1) & 0xFFFFFFFF, (right | p) >> 1
        else:
            out.append((cur, left, right, depth | 2 << 8))
    return np.array(out, dtype=np.uint32).view(_lib.SUB_DTYPE).reshape(-1)


def test_wide_boards_n29_to_32_deep_records(oracle):
    """Bit-31 handling (bitboard.hpp:36-44): random deep records of 29..32-column
    boards (8 rows left to search), counted per record on the GPU vs the C oracle and,
    for n = 32 (check_board's upper bound, solver.hpp:45-48), vs the reference build."""
    from oracle_ctypes import Reference, reference_available
    rng = np.random.default_rng(31)
    for n in (29, 30, 31, 32):
        pick = _random_deep_records(n, n - 8, 400, rng)
        counts, high, nodes = nq.count_each(n, pick, nq.KernelVariant.lastrow, pre_rows=n - 8)
        total, want_nodes, want_counts = oracle.solve_batch(n, pick, per_sub=True)
        assert np.array_equal(counts, want_counts), n
        assert int(nodes.sum()) == want_nodes, n
        assert counts.sum() > 0, n
        rep = nq.execute_batch(n, n - 8, pick, nq.ExecuteOptions(
            config=nq.builtin_configs[0], plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 2)))
        assert rep.total == total and rep.nodes == want_nodes, n
        if n == 32 and reference_available():
            ref = Reference()
            for i in range(0, len(pick), 40):
                assert ref.count(1, 32, tuple(int(x) for x in pick[i]))[0] == int(counts[i])


def test_execute_deepens_large_frontiers_on_the_device(monkeypatch, golden):
    """nq_solve deals a coarse frontier (R-3) to the workers and deepens it on each
    device once the R-frontier passes NQB_DEVICE_EXPAND_MIN_RECORDS (default 2^20, e.g.
    N=27 R=7): same total and the same Alg. 3 node count as the host path."""
    monkeypatch.setenv("NQB_DEVICE_EXPAND_MIN_RECORDS", "1000")
    for workers in (1, 3):
        opts = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.strided, workers))
        rep = nq.execute(16, 6, opts)
        assert rep.completed and rep.total == 14772512
        assert rep.nodes == golden["appendix_b_nodes"]["16"]["6"]
        assert rep.task_count == nq.count_subproblems(16, 6)
        assert sum(w.processed for w in rep.workers) == rep.task_count
    monkeypatch.setenv("NQB_DEVICE_EXPAND_MIN_RECORDS", str(1 << 62))
    assert nq.execute(16, 6, nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.strided, 1))).total == 14772512


def test_one_worker_plans_deepen_on_the_device(monkeypatch, golden):
    """With ONE worker every strategy (the reference's default plan is weighted with one
    worker) takes the device-deepening path, and the report and log lines keep the
    reference's semantics: a range worker is assigned the whole R-frontier
    (scheduler.hpp:330, :336-340), a stealing worker 0 (:106, :350)."""
    monkeypatch.setenv("NQB_DEVICE_EXPAND_MIN_RECORDS", "1000")
    total = nq.count_subproblems(16, 6)
    for strategy in (nq.PartitionStrategy.weighted, nq.PartitionStrategy.uniform,
                     nq.PartitionStrategy.stealing):
        lines = []
        opts = nq.ExecuteOptions(plan=nq.PartitionPlan(strategy, 1, [], 64), log=lines.append)
        rep = nq.execute(16, 6, opts)
        assert rep.completed and rep.total == 14772512
        assert rep.nodes == golden["appendix_b_nodes"]["16"]["6"]
        assert rep.task_count == total and rep.workers[0].processed == total
        start = [x for x in lines if "start job" in x]
        assert len(start) == 1
        if strategy is nq.PartitionStrategy.stealing:
            assert rep.workers[0].assigned == 0 and "with 0(0.00) subproblems" in start[0]
        else:
            assert rep.workers[0].assigned == total
            assert f"with {total}(1.00) subproblems" in start[0], start[0]


def test_bench_samples_rederived_on_device():
    """The CPU-baseline slices bench.py times (tests/golden/bench_samples.json, pinned
    with the C oracle) give the same weighted total and node count on the GPU."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_samples.json")) as f:
        samples = json.load(f)
    c = Ctx()
    for key, want in samples.items():
        n, r, stride = map(int, key.split(","))
        sl = nq.generate_slice(n, r, stride, 0)
        assert len(sl) == want["records"], key
        res = c.count(n, r, sl)
        assert (res.solutions, res.nodes) == (want["total"], want["nodes"]), key
    c.close()


def test_context_refuses_a_second_launch_while_one_is_in_flight(oracle):
    import torch
    a = oracle.generate(16, 5)
    dev = torch.from_numpy(a.view(np.int32).reshape(-1, 4)).cuda()
    c = Ctx()
    _lib.check(_lib.lib.nq_count_device_async(c.p, 16, 5, _lib.VARIANT_LASTROW,
                                              ctypes.c_void_p(dev.data_ptr()), len(a)))
    with pytest.raises(_lib.NqError) as e:
        c.count(16, 5, a)
    assert "in flight" in str(e.value)
    r = _lib.NqResult()
    _lib.check(_lib.lib.nq_collect(c.p, ctypes.byref(r)))
    assert r.solutions == 14772512
    assert c.count(16, 5, a).solutions == 14772512
    c.close()


def test_report_json_consistent_totals():
    """test_scheduler.cpp:149-163: the report serialises with per-worker partial sums
    that add up to the total."""
    opts = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.weighted, 4, [0.4, 0.3, 0.2, 0.1]))
    rep = nq.execute(10, 2, opts)
    j = rep.to_json()
    assert j["n"] == 10 and j["total"] == rep.total == 724
    assert len(j["workers"]) == 4 and j["partition"] == "weighted"
    assert sum(w["partial_sum"] for w in j["workers"]) == rep.total


def test_tail_donation_keeps_every_count_and_balances(golden):
    """Intra-warp donation splits subtrees between lanes at the end of a launch: the
    weighted total, raw total, node count and record count are unchanged — on a
    maximally skewed input (N=18 from R=3: 36 huge subtrees for ~150k lanes, so
    nearly all the work is donated) and on a full frontier."""
    for n, r in ((18, 3), (17, 6)):
        recs = nq.generate_packed(n, r)
        outs = []
        for balance in (0, 1):
            c = Ctx(balance=balance)
            res = c.count(n, r, recs)
            c.close()
            outs.append((res.solutions, res.raw_solutions, res.nodes, res.subproblems, res.kernel_ms))
        assert outs[0][:4] == outs[1][:4], outs
        assert outs[1][0] == golden["oeis_a000170"][n - 1]
        if r == 3:  # a from-the-root split: Alg. 3 nodes from R=3 = R=5 count + rows 4, 5
            want = golden["appendix_b_nodes"]["18"]["5"] + nq.count_subproblems(18, 4) + nq.count_subproblems(18, 5)
            assert outs[1][2] == want


def test_deepening_through_an_all_dead_level():
    """A root whose next level has records but whose level after that has none (n=5, two
    rows placed): deepening to 4 rows yields zero records, and counting through the
    deepening paths returns 0 instead of launching empty grids (round-1 ADVICE)."""
    import torch
    root = np.array([(17, 36, 8, 514)], dtype=np.uint32).view(_lib.SUB_DTYPE).reshape(-1)
    assert len(nq.expand(5, root, 3)) == 1 and len(nq.expand(5, root, 4)) == 0
    dev = torch.from_numpy(root.view(np.int32).reshape(-1, 4)).cuda()
    total = ctypes.c_uint64()
    _lib.check(_lib.lib.nq_expand_device(0, 5, ctypes.c_void_p(dev.data_ptr()), 1, 4, None, 0,
                                         ctypes.byref(total)))
    assert total.value == 0
    c = Ctx()
    r = _lib.NqResult()
    _lib.check(_lib.lib.nq_count_expand(c.p, 5, 4, _lib.VARIANT_LASTROW, root.ctypes.data, 1,
                                        ctypes.byref(r)))
    assert r.solutions == 0 and r.subproblems == 0
    c.close()
    for strategy in (nq.PartitionStrategy.strided, nq.PartitionStrategy.guided):
        rep = nq.execute_batch_expand(5, 4, root, nq.ExecuteOptions(
            config=CFG1, plan=nq.PartitionPlan(strategy, 2)))
        assert rep.total == 0 and rep.completed

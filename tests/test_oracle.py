"""Pin the C oracle (oracle/nq_oracle.c) before trusting it as the GPU checker.

Against: the golden vectors recorded from the reference itself (tests/golden/, made by
tests/golden/make_golden.py from oracle/_ref/libnqref.so), the reference's own test
assertions restated (test_solver.cpp, test_subproblems.cpp, test_scheduler.cpp,
test_bitboard.cpp), OEIS A000170, and — where this container has /root/reference — the
live reference build.
"""
import io
import numpy as np
import pytest

from oracle_ctypes import SUB_DTYPE, OracleError, Reference, reference_available


def as_recs(lst):
    return np.array([tuple(r) for r in lst], dtype=SUB_DTYPE)


def test_generate_matches_reference_records(oracle, golden):
    for key, rows in golden["generate"].items():
        n, r = map(int, key.split(","))
        got = oracle.generate(n, r)
        assert got.tolist() == [tuple(x) for x in rows], key


def test_count_subproblems_matches_reference(oracle, golden):
    for key, size in golden["count_subproblems"].items():
        n, r = map(int, key.split(","))
        if n > 22:
            continue  # the C recursion is slow-ish above; 27/7 is pinned below
        assert oracle.count_subproblems(n, r) == size, key


def test_subcount_27_7_anchor(oracle, golden):
    # acceptance.cpp:77-89
    assert golden["count_subproblems"]["27,7"] == 453688251
    assert oracle.count_subproblems(27, 7) == 453688251


def test_per_subproblem_counts_and_high_water(oracle, golden):
    # test_solver.cpp:70-80, :92-103, :116-134 — every subproblem, both kernels
    for key, d in golden["per_subproblem"].items():
        n, _ = map(int, key.split(","))
        for rec, it, lr, rc in zip(d["records"], d["iterative"], d["lastrow"], d["recursive"]):
            assert list(oracle.count_iterative(n, tuple(rec))) == it, (key, rec)
            c, h, _ = oracle.count_lastrow(n, tuple(rec))
            assert [c, h] == lr, (key, rec)
            assert oracle.count_recursive(n, rec[0], rec[1], rec[2]) == rc


def test_q_of_n_matches_oeis(oracle, golden):
    for n in range(2, 14):
        r = min(6, n - 1)
        total, _ = oracle.solve_batch(n, oracle.generate(n, r), threads=4)
        assert total == golden["oeis_a000170"][n - 1]
        assert total == golden["execute_totals"][str(n)]["total"]


def test_trivial_boards():
    # test_solver.cpp:59-63
    from oracle_ctypes import Oracle
    o = Oracle()
    assert o.count_recursive(1, 0, 0, 0) == 1
    assert o.count_recursive(2, 0, 0, 0) == 0
    assert o.count_recursive(3, 0, 0, 0) == 0
    assert o.count_lastrow(4, (0, 0, 0, 0))[0] == 2  # test_solver.cpp:93


@pytest.mark.parametrize("n", [14, 15])
def test_node_counts_appendix_b(oracle, golden, n):
    for r, nodes in golden["appendix_b_nodes"][str(n)].items():
        total, got = oracle.solve_batch(n, oracle.generate(n, int(r)))
        assert got == nodes
        assert total == golden["oeis_a000170"][n - 1]


def test_infeasible_depth_message(oracle):
    # test_solver.cpp:42-57: depth 14 > config5's 6; config3 (16) is the smallest fit
    with pytest.raises(OracleError) as e:
        oracle.count_iterative(14, (0, 0, 0, 0), depth=6)
    assert "smallest sufficient config is 'config3'" in str(e.value)


def test_aggregate_semantics(oracle):
    a = oracle.generate(5, 1)
    counts = [oracle.count_recursive(5, int(r["cols"]), int(r["diag"]), int(r["antidiag"])) for r in a]
    assert oracle.aggregate(a, counts) == 10  # test_subproblems.cpp:247-254
    dup = np.concatenate([a, a[:1]])
    with pytest.raises(OracleError) as e:
        oracle.aggregate(dup, counts + counts[:1])
    assert e.value.code == -2
    huge = np.array([(1, 2, 0, 1 | (2 << 8))], dtype=SUB_DTYPE)
    with pytest.raises(OracleError) as e:
        oracle.aggregate(huge, [2**63])
    assert e.value.code == -3


def test_partitions(oracle):
    # test_scheduler.cpp:27-62
    assert [b - a for a, b in oracle.partition_uniform(10, 4)] == [3, 3, 2, 2]
    w = [0.20, 0.15, 0.12, 0.11, 0.11, 0.11, 0.10, 0.10]
    assert [b - a for a, b in oracle.partition_weighted(100, w)] == [20, 15, 12, 11, 11, 11, 10, 10]
    first = oracle.partition_weighted(453688251, w)[0]
    assert 90737650 <= first[1] - first[0] <= 90737651
    with pytest.raises(OracleError):
        oracle.partition_weighted(10, [0.5, 0.0])


@pytest.mark.skipif(not reference_available(), reason="reference build not present")
def test_oracle_matches_reference_build_random(oracle):
    """Random legal roots at n=10..13 through the live reference build and the oracle."""
    ref = Reference()
    rng = np.random.default_rng(2511)
    for n in (10, 11, 12, 13):
        a = ref.generate(n, 3)
        for i in rng.choice(len(a), size=min(60, len(a)), replace=False):
            rec = tuple(int(x) for x in a[i])
            assert ref.count(1, n, rec) == oracle.count_lastrow(n, rec)[:2]
            assert ref.count(0, n, rec) == oracle.count_iterative(n, rec)


@pytest.mark.skipif(not reference_available(), reason="reference build not present")
def test_reference_execute_batch_threads():
    ref = Reference()
    a = ref.generate(12, 4)
    for strategy in (0, 1, 2):
        for workers in (1, 3, 8):
            total, _, processed = ref.execute_batch(12, 4, a, workers=workers, chunk=3,
                                                    strategy=strategy)
            assert total == 14200 and processed == len(a)

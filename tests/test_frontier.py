"""The PRODUCT frontier generator (libnqb200.so, host C++) vs the reference's stream.

No GPU needed: generation is host code. Mirrors test_subproblems.cpp and
acceptance.cpp criterion 2 (subcount 27 7).
"""
import io
import re

import numpy as np
import pytest

from paper_2511_12009_b200 import nqueens as nq


def test_generate_records_bit_exact(golden):
    for key, rows in golden["generate"].items():
        n, r = map(int, key.split(","))
        got = nq.generate_packed(n, r)
        assert got.tolist() == [tuple(x) for x in rows], key


def test_generate_matches_oracle_medium(oracle):
    for n, r in [(14, 4), (16, 5), (17, 6), (19, 3), (20, 6), (21, 2)]:
        a = nq.generate_packed(n, r)
        b = oracle.generate(n, r)
        assert a.shape == b.shape and np.array_equal(a, b), (n, r)


def test_count_subproblems_table(golden):
    for key, size in golden["count_subproblems"].items():
        n, r = map(int, key.split(","))
        assert nq.count_subproblems(n, r) == size, key


def test_subcount_27_7():
    # acceptance.cpp:77-89; PAPER.md:440 (453,688,251 generated in 9,287.60 ms there)
    assert nq.count_subproblems(27, 7) == 453688251


def test_n5_roots():
    # test_subproblems.cpp:34-44
    b = nq.generate(nq.GenerationPlan(5, 1))
    assert [s.cur for s in b] == [0b00001, 0b00010, 0b00100]
    assert [s.multiplier for s in b] == [2, 2, 1]
    assert all(s.placed_rows == 1 for s in b)


def test_invariants_and_determinism():
    # test_subproblems.cpp:63-78
    for n in (6, 9, 11):
        for r in (1, 2, 3):
            a = nq.generate_packed(n, r)
            cols = a["cols"]
            assert all(bin(int(c)).count("1") == r for c in cols)
            mult = a["row"] >> 8
            assert set(mult.tolist()) <= {1, 2}
            if n % 2 == 0 or r > 1:
                assert (mult == 2).all()
            keys = set(zip(a["cols"].tolist(), a["diag"].tolist(), a["antidiag"].tolist()))
            assert len(keys) == len(a)
            assert np.array_equal(a, nq.generate_packed(n, r))


def test_slices_partition_the_stream():
    full = nq.generate_packed(18, 5)
    for stride, offset in [(7, 0), (7, 3), (10000, 0), (1, 0), (3, 2)]:
        s = nq.generate_slice(18, 5, stride, offset)
        assert np.array_equal(s, full[offset::stride]), (stride, offset)


def test_plan_validation():
    # test_subproblems.cpp:126-132
    for n, r in [(5, 0), (5, 5), (1, 1), (12, 9), (40, 2)]:
        with pytest.raises(nq.ConfigError):
            nq.generate_packed(n, r)


def test_write_batch_bytes(golden):
    # test_subproblems.cpp:134-150
    for key, text in golden["write_batch"].items():
        n, r = map(int, key.split(","))
        out = io.StringIO()
        lines = nq.write_batch(out, nq.GenerationPlan(n, r))
        assert out.getvalue() == text
        assert lines == text.count("\n")
    out = io.StringIO()
    nq.write_batch(out, nq.GenerationPlan(5, 1))
    assert out.getvalue() == "0 1 2 0 1 2\n1 2 4 1 1 2\n2 4 8 2 1 1\n"


def test_aggregate_mirror():
    b = nq.generate(nq.GenerationPlan(5, 1))
    counts = [2, 4, 2]  # per-root completions of the 5x5 board
    assert nq.aggregate(list(zip(b, counts))) == 2 * 2 + 2 * 4 + 1 * 2
    with pytest.raises(nq.ConfigError):
        nq.aggregate(list(zip(b + b[:1], counts + counts[:1])))
    with pytest.raises(OverflowError):
        nq.aggregate([(nq.Subproblem(1, 2, 0, 1, 2), 2**63)])


def test_expand_reproduces_deeper_frontier():
    """nq_expand of the R-frontier to depth R' is the R'-frontier, record for record
    (the reference stream is a DFS, so deepening each root in order preserves it)."""
    for n, r0, r1 in ((9, 2, 5), (12, 4, 7), (13, 2, 6), (15, 5, 8)):  # r0 >= 2: odd-N centre fold
        got = nq.expand(n, nq.generate_packed(n, r0), r1)
        assert np.array_equal(got, nq.generate_packed(n, r1)), (n, r0, r1)
    a = nq.generate_packed(11, 6)
    assert np.array_equal(nq.expand(11, a, 4), a)  # already deep enough: copied
    assert len(nq.expand(11, a[:0], 8)) == 0
    bad = a[:3].copy()
    bad["row"][1] += 1  # popcount(cols) != placed_rows
    with pytest.raises(nq.ConfigError):
        nq.expand(11, bad, 8)

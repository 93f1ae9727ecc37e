"""Property-based checks (hypothesis) of the host-side pieces of the path: the folded
frontier generator, its slices and deepening, and the partition arithmetic — all
against the C oracle / plain-Python restatements, no GPU needed."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2511_12009_b200 import nqueens as nq


@settings(max_examples=60, deadline=None)
@given(n=st.integers(4, 13), r=st.integers(1, 6), stride=st.integers(1, 9), offset=st.integers(0, 9))
def test_slice_is_a_stride_of_the_stream(oracle, n, r, stride, offset):
    if r >= n:
        return
    full = oracle.generate(n, r)
    assert np.array_equal(nq.generate_slice(n, r, stride, offset), full[offset::stride])
    assert nq.count_subproblems(n, r) == len(full)


@settings(max_examples=40, deadline=None)
@given(n=st.integers(5, 13), r0=st.integers(2, 5), extra=st.integers(0, 4))
def test_deepening_composes(oracle, n, r0, extra):
    r1 = r0 + extra
    if r1 >= n or r1 > 8:  # the reference generator caps R at 8 (subproblems.hpp:37-38)
        return
    assert np.array_equal(nq.expand(n, oracle.generate(n, r0), r1), oracle.generate(n, r1))


@settings(max_examples=200, deadline=None)
@given(tasks=st.integers(0, 10**7), weights=st.lists(st.floats(0.01, 5.0), min_size=1, max_size=16))
def test_partitions_cover_in_order(tasks, weights):
    for ranges in (nq.partition_uniform(tasks, len(weights)), nq.partition_weighted(tasks, weights)):
        at = 0
        for r in ranges:
            assert r.first == at and r.last >= r.first
            at = r.last
        assert at == tasks
    u = nq.partition_uniform(tasks, len(weights))
    sizes = [r.size() for r in u]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)

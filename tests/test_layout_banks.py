"""Layout self-check: the DFS kernel's actual shared-memory address
functions fed to the reference's analytical bank model (bankmodel.hpp:62-99, restated
below as test code), for warps whose lanes sit at arbitrary, different stack depths —
the situation the interleaved layout must survive. The restatement is pinned to the
reference's compiled bankmodel.hpp (oracle/_ref, nqref_conflict_degree) on random
requests and on the reference's own test anchors (test_bankmodel.cpp:20-99); ncu checks
the device (profiles/)."""
import random

import pytest

BANKS, WORD = 32, 4


def conflict_degree(addresses, width, quarter=True, lanes=None):
    """bankmodel.hpp:62-99: transactions and worst per-bank degree; 16-byte accesses run
    as quarter-warp phases; identical words broadcast. `lanes` (an extension for
    predicated accesses) assigns each address to the quarter-warp of its lane id instead
    of its position in the list."""
    if not addresses:
        return 0, 0
    if lanes is not None and width == 16:
        trans = worst = 0
        for q in range(4):
            sub = [a for a, l in zip(addresses, lanes) if l // 8 == q]
            if sub:
                t, w = conflict_degree(sub, 16, quarter=False)
                trans += t
                worst = max(worst, w)
        return trans, worst
    if width == 4:
        per = {}
        for a in addresses:
            per.setdefault((a // WORD) % BANKS, set()).add(a // WORD)
        d = max(len(s) for s in per.values())
        return d, d
    phase = 8 if quarter else len(addresses)
    trans = worst = 0
    for b in range(0, len(addresses), phase):
        per = {}
        for a in addresses[b:b + phase]:
            for k in range(4):
                w = a // WORD + k
                per.setdefault(w % BANKS, set()).add(w)
        d = max(len(s) for s in per.values())
        trans += d
        worst = max(worst, d)
    return trans, worst


# The kernel's address functions (paper_2511_12009_b200/csrc/nq_kernel.cuh), byte
# offsets from the dynamic shared-memory base.
def v4_frame(t, level, block):        # kLayoutV4: uint4 at stk[level*BLOCK + t]
    return (level * block + t) * 16


def plane_word(t, level, w, block):   # kLayoutPlanes: u32 at ((4*level + w)*BLOCK + t)
    return ((4 * level + w) * block + t) * 4


@pytest.mark.parametrize("block", [64, 96, 128, 192, 256])
def test_v4_frames_conflict_free_at_any_depth_mix(block):
    rng = random.Random(block)
    for warp in range(block // 32):
        for _ in range(300):
            levels = [rng.randrange(20) for _ in range(32)]
            addrs = [v4_frame(warp * 32 + lane, levels[lane], block) for lane in range(32)]
            trans, worst = conflict_degree(addrs, 16)
            assert worst == 1 and trans == 4


@pytest.mark.parametrize("block", [64, 128, 256])
def test_planes_conflict_free_for_any_active_subset(block):
    rng = random.Random(block + 1)
    for _ in range(300):
        levels = [rng.randrange(20) for _ in range(32)]
        active = [lane for lane in range(32) if rng.random() < 0.37] or [0]
        for w in range(4):
            addrs = [plane_word(lane, levels[lane], w, block) for lane in active]
            assert conflict_degree(addrs, 4) == (1, 1)


def test_block_sizes_not_multiple_of_8_conflict():
    """Why BLOCK is restricted to multiples of 32: with a level stride
    of 100 frames, lanes at different depths collide within a quarter-warp."""
    rng = random.Random(7)
    worst = max(conflict_degree([v4_frame(l, rng.randrange(20), 100) for l in range(32)], 16)[1]
                for _ in range(200))
    assert worst >= 2


def test_sparse_v4_phases_match_hardware():
    """Lanes 0 and 8 (same bank group, different quarter-warps): two phases of degree 1 —
    two wavefronts, as tools/microbench/smem_banks.cu measures on the B200 (ncu reports
    the second as a 'conflict' against an ideal of one)."""
    assert conflict_degree([v4_frame(0, 3, 128), v4_frame(8, 5, 128)], 16, lanes=[0, 8]) == (2, 1)
    assert conflict_degree([v4_frame(0, 3, 128), v4_frame(1, 5, 128)], 16, lanes=[0, 1]) == (1, 1)


# ---- pinned to the reference's own model (bankmodel.hpp compiled in oracle/_ref) ----------
ref_only = pytest.mark.skipif(not __import__("oracle_ctypes").reference_available(),
                              reason="oracle/_ref/libnqref.so (reference build) not present")


@ref_only
def test_restatement_equals_reference_bankmodel_on_random_requests():
    """conflict_degree above == nqueens::conflict_degree (bankmodel.hpp:62-99) for random
    scalar and 16-byte requests of 1..32 threads, both warp schedules."""
    from oracle_ctypes import Reference
    ref = Reference()
    rng = random.Random(2511)
    for trial in range(3000):
        width = 4 if trial % 2 else 16
        threads = rng.randrange(1, 33)
        span = rng.choice([64, 512, 4096])
        addrs = [rng.randrange(span) * width for _ in range(threads)]
        for quarter in (True, False):
            assert conflict_degree(addrs, width, quarter=quarter) == \
                ref.conflict_degree(addrs, width, full_warp=not quarter), (addrs, width, quarter)


@ref_only
def test_reference_anchor_cases():
    """The reference's own test anchors (test_bankmodel.cpp:20-99) through both models."""
    from oracle_ctypes import Reference
    ref = Reference()
    cases = [([256] * 32, 4, True, (1, 1)),                          # broadcast
             ([4 * t for t in range(32)], 4, True, (1, 1)),          # one word per bank
             ([t * 128 for t in range(32)], 4, True, (32, 32)),      # one bank, 32 words
             ([16 * t for t in range(32)], 16, True, (4, 1)),        # interleaved frames, quarters
             ([16 * t for t in range(32)], 16, False, (4, 4))]       # ... one full-warp phase
    for addrs, width, quarter, want in cases:
        assert ref.conflict_degree(addrs, width, full_warp=not quarter) == want
        assert conflict_degree(addrs, width, quarter=quarter) == want


@ref_only
def test_kernel_layouts_through_the_reference_model():
    """The kernel's actual address functions, fed to the reference's model itself: V4
    frames at any per-lane depth mix take 4 quarter-warp transactions of degree 1; every
    plane word of any active subset is one conflict-free transaction."""
    from oracle_ctypes import Reference
    ref = Reference()
    rng = random.Random(7)
    for block in (64, 128, 256):
        for _ in range(200):
            levels = [rng.randrange(20) for _ in range(32)]
            assert ref.conflict_degree([v4_frame(l, levels[l], block) for l in range(32)], 16) == (4, 1)
            active = [l for l in range(32) if rng.random() < 0.37] or [0]
            for w in range(4):
                assert ref.conflict_degree([plane_word(l, levels[l], w, block) for l in active], 4) == (1, 1)

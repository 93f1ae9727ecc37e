"""Layout self-check: the DFS kernel's actual shared-memory address
functions fed to the reference's analytical bank model (bankmodel.hpp:62-99, restated
below as test code), for warps whose lanes sit at arbitrary, different stack depths —
the situation the interleaved layout must survive. ncu confirms on the device
(profiles/r01_ncu_dfs_*_n18.md)."""
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

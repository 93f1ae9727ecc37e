"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/nq_gpu.h declares, and its host-side logic (partitions, log lines, errors,
feasibility) behaves like the reference's (test_scheduler.cpp, test_solver.cpp)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2511_12009_b200 import nqueens as nq
from paper_2511_12009_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(REPO, "include", "nq_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nq_[a-z0-9_]+)\s*\(", src)) - {"nq_log_fn"})


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (nq_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_abi_version():
    assert _lib.lib.nq_abi_version() == 2  # 2: nq_dispatch_*, solve_batch_device, span_ms


def test_partitions_like_reference():
    sizes = [r.size() for r in nq.partition_uniform(10, 4)]
    assert sizes == [3, 3, 2, 2]
    assert all(r.size() == 1 for r in nq.partition_uniform(8, 8))
    sizes = [r.size() for r in nq.partition_weighted(100, nq.paper_gpu_weights)]
    assert sizes == [20, 15, 12, 11, 11, 11, 10, 10]
    rs = nq.partition_weighted(453688251, nq.paper_gpu_weights)
    assert 90737650 <= rs[0].size() <= 90737651
    assert rs[-1].last == 453688251
    assert nq.partition_weighted(7, [1.0])[0].size() == 7
    with pytest.raises(nq.ConfigError):
        nq.partition_uniform(10, 0)
    for bad in ([0.5, 0.0], [0.5, -0.1], []):
        with pytest.raises(nq.ConfigError):
            nq.partition_weighted(10, bad)


def test_random_partitions_cover(oracle):
    import numpy as np
    rng = np.random.default_rng(7)
    for _ in range(300):
        tasks = int(rng.integers(0, 100000))
        workers = int(rng.integers(1, 17))
        got = [(r.first, r.last) for r in nq.partition_uniform(tasks, workers)]
        assert got == oracle.partition_uniform(tasks, workers)
        w = (0.01 + rng.integers(0, 1000, size=workers) / 1000.0).tolist()
        got = [(r.first, r.last) for r in nq.partition_weighted(tasks, w)]
        assert got == oracle.partition_weighted(tasks, w)


def test_log_lines():
    # test_scheduler.cpp:132-147
    ts = re.compile(r"^\[\d{4}-\d{2}-\d{2} \d{2}:\d{2}:\d{2}\.\d{3}\] ")
    g = nq.log_generation_line(9287.6, 453688251)
    assert ts.search(g) and "Use 9287.60ms to generate 453688251 subproblems!" in g
    assert "worker [0] start job, with 90737656(0.20) subproblems." in nq.log_start_line(0, 90737656, 0.20)
    assert "worker [3] finish job." in nq.log_finish_line(3)
    res = re.compile(r"n (\d+) queens result (\d+), calc time: \[([0-9.]+) ms\]")
    m = res.search(nq.log_result_line(27, 234907967154122528, 12.5))
    assert m and m.group(2) == "234907967154122528"


def test_stack_configs_table():
    # test_solver.cpp:16-40
    rows = [("config1", 128, 96, 24, 30), ("config2", 160, 76, 19, 25), ("config3", 192, 64, 16, 22),
            ("config4", 256, 48, 12, 18), ("config5", 512, 24, 6, 12)]
    assert len(nq.builtin_configs) == 5
    for name, block, words, depth, max_n in rows:
        c = nq.find_config(name)
        assert (c.block_size, c.stack_words, c.max_depth(), c.max_n()) == (block, words, depth, max_n)


def test_require_feasible_message():
    # test_solver.cpp:42-57 (raised before any device work)
    with pytest.raises(nq.ConfigError) as e:
        nq.count_iterative(14, nq.Subproblem(), nq.find_config("config5"))
    assert "smallest sufficient config is 'config3'" in str(e.value)
    with pytest.raises(nq.ConfigError):
        nq.count_recursive(0, nq.Subproblem())
    with pytest.raises(nq.ConfigError):
        nq.count_recursive(33, nq.Subproblem())


def test_checked_arithmetic():
    # test_solver.cpp:144-149
    with pytest.raises(OverflowError):
        nq.checked_add(2**64 - 1, 1)
    with pytest.raises(OverflowError):
        nq.checked_mul(2**64 - 1, 2)
    assert nq.checked_add(2, 3) == 5 and nq.checked_mul(2, 3) == 6


def test_bitboard_helpers():
    # test_bitboard.cpp:13-17, :41-51, :92-95
    assert nq.valid_positions(0, 0, 0, 5) == 0b11111
    assert nq.valid_positions(0b00001, 0b00010, 0, 5) == 0b11100
    assert nq.valid_positions(nq.board_mask(5), 0, 0, 5) == 0
    s = nq.apply_placement(0b00001, 0b00010, 0, 0b00100)
    assert (s.cur, s.left, s.right) == (0b00101, 0b01100, 0b00010)
    assert nq.apply_placement(0, 0x80000000, 0, 1).left == 2


def test_execute_rejects_bad_options_before_device_work():
    opts = nq.ExecuteOptions()
    opts.plan = nq.PartitionPlan(nq.PartitionStrategy.uniform, 2)
    opts.config = nq.find_config("config5")  # depth 6 < 13 - 2 - 1 (test_scheduler.cpp:165-171)
    with pytest.raises(nq.ConfigError):
        nq.execute_batch(13, 2, nq.generate_packed(13, 2), opts)
    opts = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.stealing, 2, [], 0))
    with pytest.raises(nq.ConfigError):
        nq.execute_batch(8, 2, nq.generate_packed(8, 2), opts)
    with pytest.raises(nq.ConfigError):
        nq.partition_strategy_from("roundrobin")


def test_header_is_plain_c_and_links(tmp_path):
    """include/nq_gpu.h compiles as strict C99 and a C program links libnqb200.so —
    the boundary a cgo / JNI / ctypes binding sees."""
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "c_abi.c"
    src.write_text('#include "nq_gpu.h"\n'
                   "int main(void) { nq_result r; nq_solve_opts o = {0}; uint64_t t = 0;\n"
                   "  (void)r; (void)o;\n"
                   "  if (nq_count_subproblems(27, 7, &t) != NQ_OK || t != 453688251ull) return 2;\n"
                   "  if (nq_count_subproblems(5, 9, &t) != NQ_ECONFIG) return 3;\n"
                   "  return nq_abi_version() == NQ_ABI_VERSION ? 0 : 4; }\n")
    exe = tmp_path / "c_abi"
    lib_dir = os.path.join(repo, "paper_2511_12009_b200")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror",
                    "-I" + os.path.join(repo, "include"), str(src), "-L" + lib_dir, "-l:libnqb200.so",
                    "-Wl,-rpath," + lib_dir, "-o", str(exe)], check=True)
    assert subprocess.run([str(exe)]).returncode == 0

"""The reference-style CLI (paper_2511_12009_b200/cli.py): host-side subcommands and the
exit-code mapping of tools/nqueens_cli.cpp:28-31, :391-402."""
import re
import subprocess
import sys

import pytest


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2511_12009_b200.cli", *args],
                          capture_output=True, text=True, timeout=300)


def test_subcount_27_7_log_line():
    out = run("subcount", "--n", "27", "--pre-rows", "7")
    assert out.returncode == 0
    assert re.search(r"^\[\d{4}-\d\d-\d\d \d\d:\d\d:\d\d\.\d{3}\] Use [0-9.]+ms to generate 453688251 subproblems!$",
                     out.stdout.strip())


@pytest.mark.parametrize("args", [
    ("solve", "--n", "8", "--pre-rows", "9"),
    ("solve", "--n", "10", "--config", "config9"),
    ("solve", "--n", "10", "--kernel", "fast"),
    ("solve", "--n", "10", "--partition", "random"),
    ("solve", "--n", "22", "--pre-rows", "2", "--config", "config5"),
    ("solve",),
])
def test_config_errors_exit_2(args):
    assert run(*args).returncode == 2


@pytest.mark.gpu
def test_solve_log_and_json():
    out = run("solve", "--n", "12", "--pre-rows", "4", "--workers", "2")
    assert out.returncode == 0
    assert re.search(r"n 12 queens result 14200, calc time: \[[0-9.]+ ms\]", out.stdout)
    js = run("solve", "--n", "11", "--format", "json")
    assert js.returncode == 0 and '"total": 2680' in js.stdout


@pytest.mark.gpu
def test_time_limit_does_not_delay_a_finished_run(tmp_path):
    """A checkpointed solve that finishes well inside --time-limit-s exits at once (the
    limit timer is a daemon and is cancelled on return), with the completed total."""
    import time
    t0 = time.monotonic()
    out = run("solve", "--n", "14", "--pre-rows", "4", "--checkpoint", str(tmp_path / "q14.ckpt"),
              "--time-limit-s", "240", "--format", "json")
    assert out.returncode == 0, out.stderr
    assert '"total": 365596' in out.stdout and '"completed": true' in out.stdout
    assert time.monotonic() - t0 < 120


def test_resume_of_bad_checkpoint_exits_4(tmp_path):
    p = tmp_path / "bad.ckpt"
    p.write_text("nqb200-checkpoint 1\nchecksum 0\n")
    assert run("resume", str(p)).returncode == 4
    assert run("solve", "--n", "12", "--checkpoint", str(p), "--resume").returncode == 4


def test_criterion_9_q27_reference_constant():
    """acceptance.cpp:234-239: the 27-queens total is kept as a named constant."""
    from paper_2511_12009_b200 import nqueens as nq
    assert nq.kQueens27Reference == 234907967154122528


@pytest.mark.gpu
def test_criterion_10_growth_ratio_via_bench():
    """acceptance.cpp:241-285: `bench` reports Q(n)/Q(n-1) > 1 for n = 10..15."""
    out = run("bench", "--n-min", "9", "--n-max", "15", "--r-min", "2", "--r-max", "2", "--reps", "1")
    assert out.returncode == 0
    lines = out.stdout.strip().splitlines()
    assert lines[0] == "n,r,config,kernel,reps,median_ms,total,ratio"
    rows = [l.split(",") for l in lines[1:]]
    assert len(rows) == 7
    for i, cells in enumerate(rows):
        assert len(cells) == 8
        if i:
            assert float(cells[7]) > 1.0
    assert [int(c[6]) for c in rows] == [352, 724, 2680, 14200, 73712, 365596, 2279184]

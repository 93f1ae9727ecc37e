"""Chunk-granular checkpoint / resume (nq_solve_checkpointed), after the reference's
test_checkpoint.cpp: round trip, checksum corruption, identity mismatch, completed
resume, and racing-cancel fault injection whose resumed total equals a clean run."""
import os
import random
import threading

import pytest

from paper_2511_12009_b200 import nqueens as nq


def fnv1a(data: bytes) -> str:
    h = 0xcbf29ce484222325
    for c in data:
        h = ((h ^ c) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def write_ckpt(path, n, r, variant, chunk, tasks, done):
    chunks = (tasks + chunk - 1) // chunk
    ident = fnv1a(f"gen-v1|{n}|{r}|{variant}|{chunk}|{tasks}".encode())
    body = f"nqb200-checkpoint 1\nidentity {ident}\nrun {n} {r} {variant} {chunk} {tasks} {chunks}\n"
    body += "".join(f"done {i} {s} {nodes}\n" for i, (s, nodes) in sorted(done.items()))
    with open(path, "w") as f:
        f.write(body + f"checksum {fnv1a(body.encode())}\n")
    return chunks


def test_completed_checkpoint_resumes_without_a_device(tmp_path):
    """Every chunk recorded: resume reports the recorded total and touches no GPU
    (test_checkpoint.cpp:112-128)."""
    n, r = 12, 4
    tasks = nq.count_subproblems(n, r)
    chunk = 1000
    k = (tasks + chunk - 1) // chunk
    # split Q(12) = 14200 over the chunks (values are opaque to the resume logic)
    done = {i: (14200 // k + (1 if i < 14200 % k else 0), 7) for i in range(k)}
    p = tmp_path / "c.ckpt"
    write_ckpt(p, n, r, 1, chunk, tasks, done)
    assert nq.checkpoint_info(p) == (n, r, k, k)
    rep = nq.execute_checkpointed(n, r, nq.ExecuteOptions(), p, chunk=chunk, resume=True)
    assert rep.completed and rep.total == 14200 and rep.nodes == 7 * k


def test_committed_n24_checkpoint_holds_q24(tmp_path):
    """runs/n24.ckpt is the file the four-call N=24 run on a B200 left behind (profiles/
    README.md). The library's own reader accepts it: the identity matches N=24, R=7, the
    lastrow kernel and chunk 9 058 722, and the checksum is valid. Resuming it needs no
    device, and its chunk sums add up to OEIS A000170(24)."""
    import shutil
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "runs", "n24.ckpt")
    p = tmp_path / "n24.ckpt"
    shutil.copy(src, p)
    assert nq.checkpoint_info(p) == (24, 7, 16, 16)
    rep = nq.execute_checkpointed(24, 7, nq.ExecuteOptions(config=nq.find_config("config1")), p,
                                  chunk=9058722, resume=True)
    assert rep.completed and rep.total == 227514171973736
    assert rep.task_count == nq.count_subproblems(24, 7) == 144939546
    assert rep.nodes == 12749488348460170


def test_corrupt_and_foreign_checkpoints_are_rejected(tmp_path):
    n, r = 12, 4
    tasks = nq.count_subproblems(n, r)
    p = tmp_path / "c.ckpt"
    write_ckpt(p, n, r, 1, 500, tasks, {0: (10, 20)})
    text = p.read_text()
    p.write_text(text.replace("done 0 10 20", "done 0 11 20"))   # payload edited
    with pytest.raises(nq.CheckpointError, match="checksum"):
        nq.execute_checkpointed(n, r, nq.ExecuteOptions(), p, resume=True)
    p.write_text(text[: len(text) // 2])                          # truncated
    with pytest.raises(nq.CheckpointError):
        nq.execute_checkpointed(n, r, nq.ExecuteOptions(), p, resume=True)
    write_ckpt(p, n, r, 1, 500, tasks, {})
    with pytest.raises(nq.CheckpointError, match="different run"):
        nq.execute_checkpointed(13, r, nq.ExecuteOptions(), p, resume=True)   # other n
    with pytest.raises(nq.CheckpointError, match="different run"):
        nq.execute_checkpointed(n, r, nq.ExecuteOptions(kernel=nq.KernelVariant.iterative), p,
                                resume=True)
    with pytest.raises(nq.CheckpointError):
        nq.execute_checkpointed(n, r, nq.ExecuteOptions(), tmp_path / "missing.ckpt", resume=True)


@pytest.mark.gpu
def test_checkpointed_run_round_trip(tmp_path):
    p = tmp_path / "run.ckpt"
    rep = nq.execute_checkpointed(16, 5, nq.ExecuteOptions(plan=nq.PartitionPlan(worker_count=2)),
                                  p, chunk=4000)
    assert rep.completed and rep.total == 14772512
    n, r, chunks, done = nq.checkpoint_info(p)
    assert (n, r) == (16, 5) and chunks == done == (70906 + 3999) // 4000
    again = nq.execute_checkpointed(16, 5, nq.ExecuteOptions(), p, resume=True)
    assert again.completed and again.total == 14772512 and again.calc_ms < rep.calc_ms + 50


@pytest.mark.gpu
def test_racing_cancel_then_resume_equals_clean_run(tmp_path):
    """acceptance.cpp:199-232 / test_checkpoint.cpp:130-169: cancel at random moments,
    resume until complete; the total is always the clean one."""
    rng = random.Random(1234)
    for trial in range(6):
        p = tmp_path / f"t{trial}.ckpt"
        rounds = 0
        resume = False
        while True:
            ev = threading.Event()
            timer = threading.Timer(rng.uniform(0.0, 0.15), ev.set)
            timer.start()
            rep = nq.execute_checkpointed(19, 6, nq.ExecuteOptions(
                cancel=ev, plan=nq.PartitionPlan(worker_count=1 + trial % 3)), p, chunk=60000,
                resume=resume)
            timer.cancel()
            rounds += 1
            resume = True
            if rep.completed:
                break
            assert rounds < 200
        assert rep.total == 4968057848, (trial, rounds)


def test_run_with_checkpoint_validation():
    """runner.hpp:52-53: stealing is refused; n == 1 short-circuits without a file."""
    spec = nq.RunSpec(12, 3, plan=nq.PartitionPlan(nq.PartitionStrategy.stealing, 2))
    with pytest.raises(nq.ConfigError, match="contiguous partition"):
        nq.run_with_checkpoint(spec, nq.CheckpointOptions("/nonexistent/x.ckpt"))
    with pytest.raises(nq.ConfigError):
        nq.run_with_checkpoint(nq.RunSpec(0, 1), nq.CheckpointOptions("x"))


@pytest.mark.gpu
def test_run_with_checkpoint_round_trip(tmp_path):
    p = str(tmp_path / "r.ckpt")
    spec = nq.RunSpec(15, 5, plan=nq.PartitionPlan(nq.PartitionStrategy.uniform, 2))
    lines = []
    rep = nq.run_with_checkpoint(spec, nq.CheckpointOptions(p, 5000), log=lines.append)
    assert rep.completed and rep.total == 2279184
    assert any("n 15 queens result 2279184" in l for l in lines)
    assert nq.run_with_checkpoint(spec, nq.CheckpointOptions(p, 5000, resume=True)).total == 2279184
    assert nq.run_with_checkpoint(nq.RunSpec(1, 0), nq.CheckpointOptions(p)).total == 1


@pytest.mark.gpu
def test_soft_stop_records_every_started_chunk(tmp_path):
    """stop_after_s: no chunk starts after the deadline, the running ones finish and are
    recorded (nothing discarded); resuming completes the count."""
    p = tmp_path / "soft.ckpt"
    first = nq.execute_checkpointed(19, 6, nq.ExecuteOptions(), p, chunk=100000, stop_after_s=0.02)
    n, r, chunks, done = nq.checkpoint_info(p)
    assert not first.completed and done < chunks
    # every chunk that started was finished and recorded — none discarded (chunks go
    # expensive end first, so the recorded ones are the `done` highest indices)
    tasks = nq.count_subproblems(19, 6)
    sizes = [min(100000, tasks - c * 100000) for c in range(chunks)]
    assert sum(w.processed for w in first.workers) == sum(sizes[chunks - done:])
    rest = nq.execute_checkpointed(19, 6, nq.ExecuteOptions(), p, chunk=100000, resume=True)
    assert rest.completed and rest.total == 4968057848


def test_cli_resume_takes_kernel_and_chunk_from_the_file(tmp_path):
    """`resume FILE` re-applies the run's kernel variant and chunk (both part of the
    file's identity): an ITERATIVE-kernel checkpoint with a custom chunk resumes, and the
    new worker / device options are accepted. Every chunk is recorded, so no GPU runs."""
    import subprocess
    import sys
    n, r, chunk = 12, 4, 700
    tasks = nq.count_subproblems(n, r)
    k = (tasks + chunk - 1) // chunk
    done = {i: (14200 // k + (1 if i < 14200 % k else 0), 3) for i in range(k)}
    p = tmp_path / "it.ckpt"
    write_ckpt(p, n, r, 0, chunk, tasks, done)
    d = nq.checkpoint_details(p)
    assert (d["kernel"], d["chunk"], d["chunks"], d["done_chunks"]) == (nq.KernelVariant.iterative, chunk, k, k)
    out = subprocess.run([sys.executable, "-m", "paper_2511_12009_b200.cli", "resume", str(p),
                          "--workers", "2", "--format", "json"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "kernel=iterative" in out.stderr and f"chunk={chunk}" in out.stderr
    assert '"total": 14200' in out.stdout

"""The drop-in C++ API (include/nqueens/*.hpp) compiled and run as a program: the
reference doctest assertions restated in tests/cpp/test_dropin.cpp."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(HERE, "cpp")
BIN = os.path.join(CPP, "test_dropin")


def _build():
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return BIN


def test_dropin_headers_host_cases():
    out = subprocess.run([_build(), "cpu"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-4000:]
    assert "0 failures" in out.stdout


@pytest.mark.gpu
def test_dropin_headers_device_cases():
    out = subprocess.run([_build(), "gpu"], capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-4000:]
    assert "0 failures" in out.stdout

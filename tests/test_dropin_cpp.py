"""The C++ drop-in headers (include/spmk/*.hpp) compiled against the product
library, running the reference's own KATs (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binary():
    from paper_2106_16064_b200 import _build

    _build.build_library(verbose=False)
    exe = _build.build_cpp_tests(verbose=False)
    assert exe and os.path.exists(exe)
    return exe


def test_dropin_host_cases(binary):
    r = subprocess.run([binary, "--host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


@pytest.mark.gpu
def test_dropin_device_cases(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout

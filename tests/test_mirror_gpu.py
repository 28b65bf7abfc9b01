"""The reference-style C++ program (tests/cpp/mirror_test.cpp) over the C++
mirror header runs on the device and passes its checks."""
from __future__ import annotations

import subprocess

import pytest

from paper_2109_00485_b200 import build


@pytest.mark.gpu
def test_cpp_mirror_program(ctx):
    binary = build.build_cpp_tests()
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout

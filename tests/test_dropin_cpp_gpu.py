"""GPU: reference-style C++ code (tests/cpp/dropin_tests.cpp, written against
#include "graphfuse/engine.hpp" & co.) compiled against the drop-in headers and
linked to libgraphfuse.so runs its checks on the B200 path."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "dropin_tests")


def test_cpp_dropin_suite(cuda):
    assert os.path.exists(BIN), "build() did not produce tests/cpp/dropin_tests"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout

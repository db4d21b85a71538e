"""The reference's OWN test suites, unmodified, against this repo's drop-in
(built by tests/cpp/build_reftests.py from /root/reference/proj sources and
the doctest shim tests/cpp/refshim/doctest.h):

* unit_tests: test_graph / test_kernels / test_schedule / test_engine /
  test_autograd / test_models (50 doctest cases) linked to libgraphfuse.so;
* acceptance: acceptance_main.cpp criteria 1-10;
* python/tests/test_smoke.py through the `graphfuse` alias package.

GPU tests: every compute call of the drop-in runs on the B200 (no CPU
fallback).  The CPU test checks the shim's SUBCASE / Approx semantics.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RT = os.path.join(ROOT, "tests", "cpp", "_reftests")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (tests/cpp/build_reftests.py needs /root/reference)")


def test_doctest_shim_semantics(tmp_path):
    exe = tmp_path / "shim_selftest"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "tests", "cpp", "refshim"),
                    os.path.join(ROOT, "tests", "cpp", "shim_selftest.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 2 | 2 passed | 0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_unit_tests(cuda):
    exe = os.path.join(RT, "unit_tests")
    _need(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-6000:])
    assert "test cases: 50 | 50 passed | 0 failed" in r.stdout, r.stderr[-6000:]
    assert r.returncode == 0


@pytest.mark.gpu
def test_reference_acceptance(cuda):
    exe = os.path.join(RT, "acceptance")
    _need(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    passed = [ln for ln in r.stdout.splitlines() if ln.startswith("[PASS] criterion")]
    assert len(passed) == 10 and r.returncode == 0, r.stdout + r.stderr[-3000:]


@pytest.mark.gpu
def test_reference_python_smoke(cuda):
    test = os.path.join(RT, "test_smoke.py")
    _need(test)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "alias"), ROOT,
                                         env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "--rootdir", RT, test], capture_output=True, text=True, timeout=900,
                       env=env, cwd=RT)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "7 passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]

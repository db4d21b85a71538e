"""Build recipe for the reference's OWN test suites against this repo's
drop-in (test infrastructure; run by __graft_entry__.build() where
/root/reference exists, outputs travel to the GPU box prebuilt).

  tests/cpp/_reftests/unit_tests   /root/reference/proj/tests/{test_main,test_graph,
                                   test_kernels,test_schedule,test_engine,
                                   test_autograd,test_models}.cpp, unmodified,
                                   compiled with the doctest shim
                                   (tests/cpp/refshim/doctest.h) against
                                   include/graphfuse + libgraphfuse.so
  tests/cpp/_reftests/acceptance   /root/reference/proj/tests/acceptance_main.cpp
  tests/cpp/_reftests/test_smoke.py  /root/reference/proj/python/tests/test_smoke.py
                                   staged unchanged (git-ignored build output,
                                   like oracle/_ref) so pytest can run it on the
                                   GPU box through the `graphfuse` alias package
                                   (tests/alias/graphfuse)

The reference's sources are only read here; nothing is copied into git.
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("GF_REFERENCE", "/root/reference/proj")
OUT = os.path.join(HERE, "_reftests")
PKG = os.path.join(ROOT, "paper_2411_16127_b200")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
UNIT = ["test_main", "test_graph", "test_kernels", "test_schedule", "test_engine",
        "test_autograd", "test_models"]


def _newer(out, deps):
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out)
                                          for d in deps)


def build(verbose=False):
    tests = os.path.join(REF, "tests")
    if not os.path.isdir(tests):
        if verbose:
            print("reference tests absent; keeping prebuilt", OUT)
        return
    os.makedirs(OUT, exist_ok=True)
    hdrs = [os.path.join(HERE, "refshim", "doctest.h"),
            os.path.join(ROOT, "include", "graphfuse", "graphfuse.hpp"),
            os.path.join(PKG, "libgraphfuse.so")]
    flags = ["-std=c++20", "-O2", f"-I{os.path.join(HERE, 'refshim')}",
             f"-I{os.path.join(ROOT, 'include')}"]
    link = [f"-L{PKG}", "-lgraphfuse", "-lgraphfuse_cuda", f"-Wl,-rpath,{PKG}",
            "-Wl,-rpath,$ORIGIN/../../../paper_2411_16127_b200"]
    jobs = [("unit_tests", [os.path.join(tests, f + ".cpp") for f in UNIT]),
            ("acceptance", [os.path.join(tests, "acceptance_main.cpp")])]
    for name, srcs in jobs:
        out = os.path.join(OUT, name)
        if _newer(out, srcs + hdrs):
            r = subprocess.run([CXX] + flags + srcs + ["-o", out] + link, capture_output=True,
                               text=True)
            if r.returncode:
                raise RuntimeError(f"reference test build failed ({name}):\n{r.stderr[-4000:]}")
    smoke = os.path.join(REF, "python", "tests", "test_smoke.py")
    if os.path.exists(smoke):
        shutil.copyfile(smoke, os.path.join(OUT, "test_smoke.py"))


if __name__ == "__main__":
    build(verbose=True)
    print("built", OUT, file=sys.stderr)

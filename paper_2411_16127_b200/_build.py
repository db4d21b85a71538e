"""In-tree build of the B200 libraries (no JIT cache; the .so files travel
with the repo snapshot to the GPU box).

  libgraphfuse_cuda.so  sm_100a kernels + the C-ABI (include/gf_cuda.h),
                        CUDA runtime linked statically, no torch.
  libgraphfuse.so       the C++ drop-in operator API (include/graphfuse/*.hpp),
                        calls only the C-ABI.
  _core.<abi>.so        pybind11 module mirroring graphfuse._core.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# The host libraries must share the process's libstdc++ (torch loads the
# system libstdc++.so): a toolchain that links libstdc++ statically (this
# image's CXX wrapper does) would export a second copy of the locale/iostream
# internals and crash std::ostream use once torch is imported.  Prefer the
# system g++; GF_CXX overrides.
CXX = os.environ.get("GF_CXX") or ("/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-Wall", "--expt-relaxed-constexpr", f"-I{INC}", f"-I{CSRC}"]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", f"-I{INC}"]

CUDA_LIB = os.path.join(PKG, "libgraphfuse_cuda.so")
HOST_LIB = os.path.join(PKG, "libgraphfuse.so")
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
CORE = os.path.join(PKG, "_core" + EXT)


def _newer(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(INC, "*.h"))
            + glob.glob(os.path.join(INC, "graphfuse", "*.hpp")))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build(verbose: bool = False) -> None:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    for src in cu:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if _newer(obj, [src] + hdrs):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj])
    host_src = sorted(glob.glob(os.path.join(CSRC, "host", "gf_host_*.cpp")))
    host_lib_src = [s for s in host_src if not s.endswith("bindings.cpp")]
    for src in host_lib_src:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if _newer(obj, [src] + hdrs):
            jobs.append([CXX] + CXX_FLAGS + ["-c", src, "-o", obj])
    if jobs:
        with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
            for r in ex.map(_run, jobs):
                if verbose and r.stderr:
                    print(r.stderr, file=sys.stderr)
    cu_obj = [os.path.join(OBJ, os.path.basename(s) + ".o") for s in cu]
    if _newer(CUDA_LIB, cu_obj):
        _run([NVCC] + ARCH + ["-shared", "-o", CUDA_LIB] + cu_obj + ["-cudart", "static"])
    host_obj = [os.path.join(OBJ, os.path.basename(s) + ".o") for s in host_lib_src]
    if _newer(HOST_LIB, host_obj + [CUDA_LIB]):
        _run([CXX, "-shared", "-o", HOST_LIB] + host_obj
             + [f"-L{PKG}", "-lgraphfuse_cuda", "-Wl,-rpath,$ORIGIN"])
    # C++ drop-in test binary: reference-style C++ code against include/graphfuse
    test_src = os.path.join(ROOT, "tests", "cpp", "dropin_tests.cpp")
    test_bin = os.path.join(ROOT, "tests", "cpp", "dropin_tests")
    if os.path.exists(test_src) and _newer(test_bin, [test_src, HOST_LIB] + hdrs):
        _run([CXX] + CXX_FLAGS + [test_src, "-o", test_bin, f"-L{PKG}", "-lgraphfuse",
                                  "-lgraphfuse_cuda", f"-Wl,-rpath,{PKG}"])
    bind = os.path.join(CSRC, "host", "gf_host_bindings.cpp")
    if _newer(CORE, [bind, HOST_LIB] + hdrs):
        import pybind11

        py_inc = sysconfig.get_paths()["include"]
        _run([CXX] + CXX_FLAGS + ["-shared", f"-I{pybind11.get_include()}", f"-I{py_inc}",
                                  "-fvisibility=hidden", bind, "-o", CORE, f"-L{PKG}",
                                  "-lgraphfuse", "-lgraphfuse_cuda", "-Wl,-rpath,$ORIGIN"])


if __name__ == "__main__":
    build(verbose=True)
    print("built:", CUDA_LIB, HOST_LIB, CORE)

"""GPU: compute-sanitizer memcheck / racecheck / synccheck over the hot
kernels (fwd_fast, bwd_rows_fast, bwd_cols_fast, the tcgen05 GEMMs) on small
graphs that exercise every schedule bucket (scripts/sanitize_small.py)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = "regex=fwd_fast|bwd_rows_fast|bwd_cols_fast|tma_gemm_kernel|tc_gemm|split_b_kernel|tn_reduce"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(cuda, tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", tool, "--error-exitcode", "3", "--kernel-name", KERNELS,
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_small.py")]
    if tool == "racecheck":
        cmd[3:3] = ["--racecheck-report", "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize workload ok" in out, out[-6000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-6000:]


def test_sanitizer_filter_instruments_named_kernels(cuda, tmp_path):
    """Negative control: the same kernel-name filter catches a deliberate
    out-of-bounds write in a kernel whose name matches it, so the clean runs
    above did instrument the hot kernels."""
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not (os.path.exists(cs) and os.path.exists(nvcc)):
        pytest.skip("compute-sanitizer / nvcc not installed")
    src = tmp_path / "negctl.cu"
    src.write_text("""
#include <cstdio>
__global__ void fwd_fast_negctl(int* p) { p[threadIdx.x + 1000000] = 1; }
int main() {
  int* p;
  cudaMalloc(&p, 64);
  fwd_fast_negctl<<<1, 32>>>(p);
  cudaDeviceSynchronize();
  printf("done\\n");
  return 0;
}
""")
    exe = tmp_path / "negctl"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", str(src), "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([cs, "--tool", "memcheck", "--error-exitcode", "3", "--kernel-name", KERNELS,
                        str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 3 and "Invalid __global__ write" in r.stdout + r.stderr, r.stdout[-3000:]

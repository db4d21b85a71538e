"""Build libgraphfuse_cuda.so with extra -D flags into variants/<name>/ for
A/B measurements (select with GF_CUDA_LIB=variants/<name>/libgraphfuse_cuda.so).

  python scripts/build_variant.py minb3 -DGF_MINB=3
"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_16127_b200 import _build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "variants", name)  # travels with gpurun (build/ does not)
    os.makedirs(out, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))
    jobs = [[B.NVCC] + B.NVCC_FLAGS + flags + ["-c", s, "-o", os.path.join(out, os.path.basename(s) + ".o")]
            for s in srcs]
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        list(ex.map(B._run, jobs))
    objs = [j[-1] for j in jobs]
    B._run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, "libgraphfuse_cuda.so")] + objs
           + ["-cudart", "static"])
    print(os.path.join(out, "libgraphfuse_cuda.so"))


if __name__ == "__main__":
    main()

"""Does tcgen05 kind::tf32 truncate fp32 inputs (ignore the low 13 mantissa
bits)?  Compare the 3xTF32 GEMM error with masked vs raw 'hi' operands."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16127_b200 import fused  # noqa: E402

rng = np.random.default_rng(0)
for M, K, N in [(4096, 128, 128), (1000, 64, 64)]:
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    C = fused.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    print(os.environ.get("GF_CUDA_LIB", "default"), M, K, N,
          "max rel", float(np.abs(C - ref).max() / np.abs(ref).max()))

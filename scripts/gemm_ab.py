"""Time one X*W shape (tcgen05 projection) — for env-override A/B runs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16127_b200 import fused  # noqa: E402

M, K, N = (int(x) for x in sys.argv[1:4])
A = torch.rand(M, K, device="cuda") * 2 - 1
B = torch.rand(K, N, device="cuda") * 2 - 1
C = torch.empty(M, N, device="cuda")
for _ in range(3):
    fused.gemm(A, B, out=C)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    fused.gemm(A, B, out=C)
b.record()
b.synchronize()
ms = a.elapsed_time(b) / 20
print(f"M{M} K{K} N{N} NT={os.environ.get('GF_TMA_NT', '-')} BRES={os.environ.get('GF_TMA_BRES', '-')}"
      f" {ms:.4f} ms {2 * M * K * N / ms / 1e9:.1f} TFLOP/s {(M * K + M * N) * 4 / ms / 1e6:.0f} GB/s")

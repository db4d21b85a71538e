"""Projection (K0) throughput: tcgen05 3xTF32 vs the SIMT fp32 kernel on the
BASELINE projection shapes.  Prints one JSON line per shape.

  python scripts/bench_gemm.py
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [  # (name, M, K, N)
    ("C4 GAT X*W (233k x 64 x 64)", 232_965, 64, 64),
    ("C5 GAT X*W (2.4M x 64 x 64)", 2_400_000, 64, 64),
    ("C5 GT X*[Wq|Wk|Wv] (2.4M x 128 x 384)", 2_400_000, 128, 384),
    ("C2 GT X*[Wq|Wk|Wv] (26.6k x 128 x 384)", 26_624, 128, 384),
]
TN_SHAPES = [  # weight gradients X^T dY: (name, K=nodes, M=F_in, N=F_out)
    ("C4 GAT dW = X^T dH (233k; 64 x 64)", 232_965, 64, 64),
    ("C5 GT dW_q = X^T dQ (2.4M; 128 x 128)", 2_400_000, 128, 128),
]


def run(simt: bool):
    import torch

    from paper_2411_16127_b200 import fused

    out = []
    for name, M, K, N in SHAPES:
        A = torch.rand(M, K, device="cuda") * 2 - 1
        B = torch.rand(K, N, device="cuda") * 2 - 1
        C = torch.empty(M, N, device="cuda")
        for _ in range(3):
            fused.gemm(A, B, out=C)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 20
        ev[0].record()
        for _ in range(reps):
            fused.gemm(A, B, out=C)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        ref = (A.double() @ B.double()).float()
        err = float(((C - ref).abs() / ref.abs().clamp_min(1.0)).max())
        out.append({"shape": name, "kernel": "simt" if simt else "tcgen05-3xtf32", "ms": ms,
                    "tflops": 2 * M * K * N / ms / 1e9, "max_rel_err": err,
                    "bytes_gbs": 4 * (M * K + K * N + M * N) / ms / 1e6})
    for name, K, M, N in TN_SHAPES:
        X = torch.rand(K, M, device="cuda") * 2 - 1
        Y = torch.rand(K, N, device="cuda") * 2 - 1
        C = torch.empty(M, N, device="cuda")
        for _ in range(3):
            fused.gemm(X, Y, trans_a=True, out=C)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            fused.gemm(X, Y, trans_a=True, out=C)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 10
        out.append({"shape": name, "kernel": "simt" if simt else "tcgen05-3xtf32-tn",
                    "ms": ms, "tflops": 2 * M * K * N / ms / 1e9,
                    "bytes_gbs": 4 * (M * K + K * N) / ms / 1e6})
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        for r in run(simt=os.environ.get("GF_GEMM_SIMT") == "1"):
            print(json.dumps(r))
    else:
        for simt in ("0", "1"):
            env = dict(os.environ, GF_GEMM_SIMT=simt)
            subprocess.run([sys.executable, __file__, "--child"], env=env, check=True)

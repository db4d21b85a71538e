"""Workload for compute-sanitizer (tests/test_gpu_sanitizer.py): the hot
kernels on small graphs, every bucket of the bi-level schedule exercised
(CTA rows and CTA columns via a low CTA threshold on a symmetric hub graph,
warp rows, packed rows, empty rows), GAT 8x8 / GT 8x16 / AGNN 1x128, the fused
forward + both backward passes, and the tcgen05 GEMMs (TMA-fed X.W,
split-K X^T.dY)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16127_b200 import fused  # noqa: E402


def graph(n=3000, hub=900, avg=4, seed=0):
    rng = np.random.default_rng(seed)
    src = np.concatenate([rng.integers(0, n, n * avg), rng.permutation(n)[:hub],
                          np.zeros(hub // 2, np.int64)])
    dst = np.concatenate([rng.integers(0, n - 200, n * avg), np.zeros(hub, np.int64),
                          rng.permutation(n)[:hub // 2]])
    key = np.unique(np.concatenate([dst * n + src]))
    s, d = torch.from_numpy(key % n).cuda(), torch.from_numpy(key // n).cuda()
    rp, col, cp, cr, _ = fused.from_coo_device(n, s, d)
    return n, fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr, cta_threshold=64)


def main():
    n, dg = graph()
    assert dg.info.n_cta_rows > 0 and dg.info.n_cta_cols > 0 and dg.info.n_empty_rows > 0
    for variant, l2, H, D in (("add", False, 8, 8), ("dot", False, 8, 16), ("dot", True, 1, 128)):
        spec = fused.AttnSpec(variant, H, D, scale=0.25, slope=0.2, l2=l2)
        w = spec.qk_width
        Q, K = torch.rand(n, w, device="cuda"), torch.rand(n, w, device="cuda")
        V, dO = torch.rand(n, H * D, device="cuda"), torch.rand(n, H * D, device="cuda")
        O, st = fused.attn_forward(dg, spec, Q, K, V)
        fused.attn_backward(dg, spec, Q, K, V, O, st, dO)
    A = torch.rand(1000, 128, device="cuda")
    B = torch.rand(128, 384, device="cuda")
    fused.gemm(A, B)
    fused.gemm(A, torch.rand(1000, 64, device="cuda"), trans_a=True)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()

"""Kernel times of the fused attention for any (variant, H, D) on a bench
graph (design probe; A/B a variant library with GF_CUDA_LIB=...).

  python scripts/probes/time_shape.py --graph reddit --variant dot --heads 8 --dim 8

Prints one line: fwd / pass A / pass B mean ms (CUDA events, cold L2 before
every launch) and GEdges/s of the three.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", default="reddit")
    ap.add_argument("--variant", default="dot", choices=("dot", "add"))
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--dim", type=int, default=8)
    ap.add_argument("--l2", action="store_true", help="AGNN-style L2-normalised dot scores")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, src, dst = bench.gen_graph_device(args.graph, dev)
    row_ptr, col, csc_ptr, csc_row, _ = fused.from_coo_device(n, src, dst)
    dg = fused.DeviceGraph.from_device_csr(n, row_ptr, col, csc_ptr, csc_row)
    e = int(src.numel())
    H, D = args.heads, args.dim
    spec = fused.AttnSpec(args.variant, H, D, scale=D ** -0.5, slope=0.2, l2=args.l2)
    w = spec.qk_width
    g = torch.Generator(device=dev).manual_seed(0)
    Q, K = (torch.rand(n, w, device=dev, generator=g) - 0.5 for _ in range(2))
    V, dO = (torch.rand(n, H * D, device=dev, generator=g) - 0.5 for _ in range(2))
    O = torch.empty(n, H * D, device=dev)
    st = torch.empty(n, H, 4, device=dev)
    dQ, dK, dV = torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ms = {"fwd": [], "bwd_rows": [], "bwd_cols": []}
    for it in range(args.iters + 2):
        for name, fn in (
            ("fwd", lambda: fused.attn_forward(dg, spec, Q, K, V, O=O, stats=st)),
            ("bwd_rows", lambda: fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK)),
            ("bwd_cols", lambda: fused.attn_backward_cols(dg, spec, Q, K, V, st, dO, dQ, dV)),
        ):
            bench.cold_l2(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                ms[name].append(a.elapsed_time(b))
    mean = {k: round(sum(v) / len(v), 4) for k, v in ms.items()}
    tot = sum(mean.values())
    print(f"{args.graph} {args.variant} {H}x{D}{' l2' if args.l2 else ''} e={e} {mean} "
          f"{e / (tot * 1e-3) / 1e9:.3f} GEdges/s "
          f"lib={os.environ.get('GF_CUDA_LIB', 'default')}", flush=True)


if __name__ == "__main__":
    main()

"""Design probe: would running backward pass A (CSR rows) and pass B (CSC
columns) concurrently beat running them back to back?  Both are gather-bound
on L2; pass A sits further from the L2 peak than pass B, so overlapping them
could fill its latency bubbles.  Pass B normally needs pass A's delta
records; the probe runs pass A once first (untimed), so the concurrent pass B
reads the same values a delta pre-pass would provide.

  python scripts/probes/overlap_ab.py [--graph reddit]
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
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, src, dst = bench.gen_graph_device(args.graph, dev)
    row_ptr, col, csc_ptr, csc_row, _ = fused.from_coo_device(n, src, dst)
    dg = fused.DeviceGraph.from_device_csr(n, row_ptr, col, csc_ptr, csc_row)
    e = int(src.numel())
    H, D = 8, 8
    spec = fused.AttnSpec("add", H, D, slope=0.2, logits_from_v=True)
    g = torch.Generator(device=dev).manual_seed(0)
    al, ar = (torch.rand(1, H * D, device=dev, generator=g) - 0.5 for _ in range(2))
    V, dO = (torch.rand(n, H * D, device=dev, generator=g) - 0.5 for _ in range(2))
    O, st = fused.attn_forward(dg, spec, al, ar, V)
    dQ, dK, dV = torch.zeros_like(al), torch.zeros_like(ar), torch.empty_like(V)
    dQ = torch.zeros(n, H, device=dev)
    dK = torch.zeros(n, H, device=dev)
    fused.attn_backward_rows(dg, spec, al, ar, V, O, st, dO, dK)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s0 = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def A(s):
        fused.attn_backward_rows(dg, spec, al, ar, V, O, st, dO, dK, stream=s)

    def B(s):
        fused.attn_backward_cols(dg, spec, al, ar, V, st, dO, dQ, dV, stream=s)

    def timed(body):
        res = []
        for it in range(args.iters + 2):
            bench.cold_l2(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s0)
            body()
            b.record(s0)
            torch.cuda.synchronize()
            if it >= 2:
                res.append(a.elapsed_time(b))
        return sum(res) / len(res)

    def seq():
        A(s0)
        B(s0)

    def conc(first, second):
        def body():
            ev = torch.cuda.Event()
            ev.record(s0)
            s1.wait_event(ev)
            s2.wait_event(ev)
            first(s1)
            second(s2)
            s0.wait_stream(s1)
            s0.wait_stream(s2)
        return body

    for rep in range(2):
        t_a = timed(lambda: A(s0))
        t_b = timed(lambda: B(s0))
        t_seq = timed(seq)
        t_ab = timed(conc(A, B))
        t_ba = timed(conc(B, A))
        print(f"{args.graph} e={e} rep {rep}: A {t_a:.4f} ms, B {t_b:.4f} ms, A;B {t_seq:.4f} ms, "
              f"A||B {t_ab:.4f} ms, B||A {t_ba:.4f} ms", flush=True)


if __name__ == "__main__":
    main()

"""Does running the heads in groups (smaller gathered footprint, higher L2 hit
rate) pay on C5 (uniform random, 2.4 M nodes)?  Times the three attention
kernels at H heads of width D for H in 8/4/2/1 and reports ms scaled to 8 heads.
Head-group launches would gather the same bytes per head from strided tables;
dense H-head tables are the proxy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402

dev = torch.device("cuda")
n, src, dst = bench.gen_graph_device("products", dev, seed=1)
rp, col, cp, cr, _ = fused.from_coo_device(n, src, dst)
del src, dst
dg = fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


for variant, D in (("dot", 16), ("add", 8)):
    for H in (8, 4, 2, 1):
        spec = fused.AttnSpec(variant, H, D, scale=0.25 if variant == "dot" else 1.0, slope=0.2)
        qk = spec.qk_width
        Q = torch.randn(n, qk, device=dev)
        K = torch.randn(n, qk, device=dev)
        V = torch.randn(n, H * D, device=dev)
        dO = torch.randn(n, H * D, device=dev)
        O, st = fused.attn_forward(dg, spec, Q, K, V)
        dQ, dK, dV = torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V)
        tf = timeit(lambda: fused.attn_forward(dg, spec, Q, K, V, O=O, stats=st))
        ta = timeit(lambda: fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK))
        tb = timeit(lambda: fused.attn_backward_cols(dg, spec, Q, K, V, st, dO, dQ, dV))
        s = 8 / H
        print(f"{variant} H={H} D={D}: fwd {tf:.3f} A {ta:.3f} B {tb:.3f} ms; x{s:g} -> "
              f"fwd {tf*s:.3f} A {ta*s:.3f} B {tb*s:.3f} total {(tf+ta+tb)*s:.3f} ms", flush=True)
        del Q, K, V, dO, O, st, dQ, dK, dV

"""Probe: pass B (CSC columns) over the whole C4 graph vs the same work split
into P destination-id ranges (one launch per range, each gathering only its
range's dO rows + records, so the gathered working set is 1/P of 90 MB).
Prints ms per variant (cold L2 before each variant's launches)."""
import os
import sys
import statistics

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402
from paper_2411_16127_b200._capi import check, lib  # noqa: E402

dev = torch.device("cuda")
check(lib().gf_l2_persist(int(os.environ.get("MIB", "64")) << 20), "persist")
n, src, dst = bench.gen_graph_device("reddit", dev)
rp, col, cp, cr, _ = fused.from_coo_device(n, src, dst)
del src, dst
dg = fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr)
spec = fused.AttnSpec("add", 8, 8, slope=0.2)
g = torch.Generator(device=dev)
g.manual_seed(1)
u = lambda *s, a=1.0: (torch.rand(*s, device=dev, generator=g) * 2 - 1) * a  # noqa: E731
Q, K, V, dO = u(n, 8, a=2.0), u(n, 8, a=2.0), u(n, 64), u(n, 64)
O, st = fused.attn_forward(dg, spec, Q, K, V)
dK = torch.empty(n, 8, device=dev)
fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK)
dQ, dV = torch.empty(n, 8, device=dev), torch.empty(n, 64, device=dev)
flush = torch.empty(64 << 20, device=dev)
col_of = torch.repeat_interleave(torch.arange(n, device=dev), cp[1:] - cp[:-1])


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        bench.cold_l2(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.mean(ts)


print("full", round(timed(lambda: fused.attn_backward_cols(dg, spec, Q, K, V, st, dO, dQ, dV)), 4))
for P in (2, 3, 4):
    graphs = []
    for k in range(P):
        lo, hi = n * k // P, n * (k + 1) // P
        m = (cr >= lo) & (cr < hi)
        crk = cr[m]
        cnt = torch.bincount(col_of[m], minlength=n)
        cpk = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        cpk[1:] = torch.cumsum(cnt, 0)
        graphs.append(fused.DeviceGraph.from_split(n, torch.zeros(n + 1, dtype=torch.int64, device=dev),
                                                   torch.zeros(1, dtype=torch.int64, device=dev), cpk,
                                                   crk, skip_empty=True))
    dVs = [torch.empty_like(dV) for _ in range(P)]

    def run():
        for k in range(P):
            fused.attn_backward_cols(graphs[k], spec, Q, K, V, st, dO, dQ, dVs[k])

    print("split", P, round(timed(run), 4))

"""Probe: cost of a der[v] scatter-reduction from a source-owned (CSC) pass
on the C4 graph, vs pass A (the destination-owned pass it would replace)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402
from paper_2411_16127_b200._capi import check, lib  # noqa: E402

L = lib()
dev = torch.device("cuda")
n, src, dst = bench.gen_graph_device("reddit", dev)
rp, col, cp, cr, _ = fused.from_coo_device(n, src, dst)
cp32, cr32 = cp.to(torch.int32), cr.to(torch.int32)
table = torch.zeros(n, 16, device=dev)
for mode, name in ((0, "red.f32 x8 lanes"), (1, "red.v4.f32 x2 lanes"), (2, "st.f32 x8 lanes"),
                   (3, "ld.f32 x8 lanes"), (4, "red.u64 x8 lanes (64 B)")):
    ms = C.c_float()
    check(L.gf_probe_scatter(n, cp32.data_ptr(), cr32.data_ptr(), table.data_ptr(), mode, 5,
                             C.byref(ms), None), "probe")
    print(f"{name}: {ms.value:.4f} ms for E={cr.numel()}")
dg = fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr)
spec = fused.AttnSpec("add", 8, 8, slope=0.2)
u = lambda *s: torch.rand(*s, device=dev) * 2 - 1  # noqa: E731
Q, K, V, dO = u(n, 8), u(n, 8), u(n, 64), u(n, 64)
O, st = fused.attn_forward(dg, spec, Q, K, V)
dK = torch.empty(n, 8, device=dev)
for i in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK)
    b.record()
    b.synchronize()
print(f"pass A: {a.elapsed_time(b):.4f} ms")

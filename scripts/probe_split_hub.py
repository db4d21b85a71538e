"""A/B of the multi-CTA split on a 200 k in/out-degree hub graph (GAT 8x8
and GT 8x16): fwd / pass A / pass B ms with the default split_len and with
splitting disabled (GF_SPLIT_LEN huge, set by the caller)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import bench  # noqa: E402
from test_gpu_parity import _mega_hub_graph  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402

g = _mega_hub_graph()
dg = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row)
flush = torch.empty(64 << 20, device="cuda")
for variant, H, D in (("add", 8, 8), ("dot", 8, 16)):
    spec = fused.AttnSpec(variant, H, D, scale=0.25)
    w = spec.qk_width
    Q, K = torch.rand(g.n, w, device="cuda"), torch.rand(g.n, w, device="cuda")
    V, dO = torch.rand(g.n, H * D, device="cuda"), torch.rand(g.n, H * D, device="cuda")
    O, st = fused.attn_forward(dg, spec, Q, K, V)
    dQ, dK, dV = (torch.empty(g.n, w, device="cuda"), torch.empty(g.n, w, device="cuda"),
                  torch.empty(g.n, H * D, device="cuda"))
    runs = {"fwd": lambda: fused.attn_forward(dg, spec, Q, K, V, O=O, stats=st),
            "bwd_rows": lambda: fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK),
            "bwd_cols": lambda: fused.attn_backward_cols(dg, spec, Q, K, V, st, dO, dQ, dV)}
    out = {}
    for k, fn in runs.items():
        ts = []
        for _ in range(6):
            bench.cold_l2(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        out[k] = round(statistics.median(ts[1:]), 4)
    print(os.environ.get("GF_SPLIT_LEN", "default"), variant, H, D, "E", g.e,
          "cta_blocks", dg.info.cta_blocks_rows, dg.info.cta_blocks_cols, out)

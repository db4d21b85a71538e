"""Per-kernel look at the unfused backward on one config (run under ncu's
launch-list mode): python scripts/profile_unfused_bwd.py [c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2411_16127_b200 import fused

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
graph, layer, H, D, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda")
n, src, dst = bench.gen_graph_device(graph, dev)
rp, col, cp, cr, _ = fused.from_coo_device(n, src, dst)
dg = fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr)
spec = fused.AttnSpec("add" if layer == "gat" else "dot", H, D,
                      scale=(1.0 / np.sqrt(D)) if layer == "gt" else 1.0, l2=layer == "agnn")
qk = spec.qk_width
Q, K = torch.rand(n, qk, device=dev), torch.rand(n, qk, device=dev)
V, dO = torch.rand(n, H * D, device=dev), torch.rand(n, H * D, device=dev)
O, st, P = fused.attn_forward(dg, spec, Q, K, V, want_p=True)
for _ in range(2):
    fused.attn_backward_unfused(dg, spec, Q, K, V, P, dO)
torch.cuda.synchronize()
print("done")

"""Fresh-process gf_measure_metrics calls (flakiness probe)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_16127_b200 import fused
from paper_2411_16127_b200._capi import GFError
x = torch.zeros(1 << 20, device="cuda")
try:
    m = fused.measure_metrics(lambda: x.add_(1), ["dram__bytes_read.sum", "dram__bytes_write.sum"])
    print("OK", m)
except GFError as e:
    print("ERR", e)

"""Gather bandwidth vs footprint and row size (gf_measure_l2_gather)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

torch.zeros(1, device="cuda")
from paper_2411_16127_b200._capi import lib  # noqa: E402

for rb in (32, 128, 256, 512):
    for mb in (32, 64, 96, 2048):
        g = C.c_double()
        rc = lib().gf_measure_l2_gather(mb << 20, rb, 5, C.byref(g), None)
        print(f"row {rb:4d} B  footprint {mb:5d} MB  rc {rc}  {g.value:8.0f} GB/s", flush=True)

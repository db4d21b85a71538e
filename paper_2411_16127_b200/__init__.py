"""B200-native fused attention-GNN layer (DF-GNN, arXiv 2411.16127).

The Python surface mirrors the reference package ``graphfuse``
(/root/reference/proj/python/graphfuse/__init__.py:3-17): same functions,
arguments, defaults and float64 semantics, served by host C++ (``_core``)
over the C-ABI of ``libgraphfuse_cuda.so`` (sm_100a kernels).  ``fused``
adds the device-resident multi-head entry points used for throughput runs.
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))


def build() -> None:
    from . import _build

    _build.build()


try:
    from ._core import (  # noqa: F401  (re-exported API, reference __init__.py:3-17)
        Graph,
        backward,
        batch_graphs,
        degree_stats,
        device_ok,
        forward,
        from_coo,
        gen_random,
        gen_super_node,
        gradcheck,
        load_graph,
        run_benchmark_json,
        save_graph,
        select_strategy,
        super_node_threshold,
    )
except ImportError as _e:  # fail loudly: there is no pure-Python / CPU fallback
    raise ImportError(
        f"paper_2411_16127_b200: compiled extension missing or broken ({_e}); run "
        "`python paper_2411_16127_b200/_build.py` (or __graft_entry__.build())") from _e

__all__ = [
    "Graph",
    "backward",
    "batch_graphs",
    "degree_stats",
    "forward",
    "from_coo",
    "gen_random",
    "gen_super_node",
    "gradcheck",
    "load_graph",
    "run_benchmark_json",
    "save_graph",
    "select_strategy",
    "super_node_threshold",
]

"""ctypes binding of the C-ABI in include/gf_cuda.h (libgraphfuse_cuda.so).

This is the same binding a maintainer would add to the reference's Python
side.  It loads the in-tree library and fails loudly if
it is missing — there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GF_CUDA_LIB overrides the library path (used only to A/B kernel build
# variants, scripts/build_variant.py); the default is the in-tree build.
LIB_PATH = os.environ.get("GF_CUDA_LIB") or os.path.join(_HERE, "libgraphfuse_cuda.so")

GF_OK = 0
GF_F32, GF_F64 = 0, 1
GF_DOT, GF_ADD = 0, 1
GF_FLAG_LOGITS_FROM_V = 1  # gf_attn_desc.reserved flag (gf_cuda.h)
GF_STRAT = {"smmf": 0, "pmf": 1, "unfused": 2, "baseline": 3}

_vp = C.c_void_p


class AttnDesc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("variant", C.c_int32), ("l2", C.c_int32),
                ("heads", C.c_int32), ("head_dim", C.c_int32), ("reserved", C.c_int32),
                ("scale", C.c_double), ("slope", C.c_double)]


class GraphInfo(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("num_edges", C.c_int64),
                ("max_in_degree", C.c_int64), ("max_out_degree", C.c_int64),
                ("cta_threshold", C.c_int32), ("n_cta_rows", C.c_int32),
                ("n_empty_rows", C.c_int32), ("n_cta_cols", C.c_int32),
                ("n_empty_cols", C.c_int32), ("device", C.c_int32),
                ("n_small_rows", C.c_int32), ("n_small_cols", C.c_int32),
                ("cta_blocks_rows", C.c_int32), ("cta_blocks_cols", C.c_int32)]


# Every symbol include/gf_cuda.h declares, with its ctypes signature.
SIGNATURES = {
    "gf_last_error": (C.c_char_p, []),
    "gf_device_ok": (C.c_int, []),
    "gf_malloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "gf_free": (C.c_int, [_vp]),
    "gf_memcpy": (C.c_int, [_vp, _vp, C.c_size_t, C.c_int32, _vp]),
    "gf_memset": (C.c_int, [_vp, C.c_int32, C.c_size_t, _vp]),
    "gf_stream_sync": (C.c_int, [_vp]),
    "gf_graph_create": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, C.c_int32, _vp,
                                  C.POINTER(_vp)]),
    "gf_graph_create_device": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, C.c_int32,
                                         _vp, C.POINTER(_vp)]),
    "gf_graph_create_split": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp,
                                        C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "gf_from_coo_device": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     C.POINTER(C.c_int64), _vp]),
    "gf_graph_destroy": (C.c_int, [_vp]),
    "gf_graph_get_info": (C.c_int, [_vp, C.POINTER(GraphInfo)]),
    "gf_graph_get_schedule": (C.c_int, [_vp, _vp, _vp]),
    "gf_attn_fwd": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gf_attn_fwd_workspace": (C.c_int, [_vp, C.POINTER(AttnDesc), C.c_int32, C.c_int32,
                                        C.POINTER(C.c_size_t)]),
    "gf_attn_fwd_strategy": (C.c_int, [_vp, C.POINTER(AttnDesc), C.c_int32, _vp, _vp, _vp, _vp,
                                       _vp, _vp, _vp, C.c_size_t, _vp]),
    "gf_time_fwd_strategy": (C.c_int, [_vp, C.POINTER(AttnDesc), C.c_int32, _vp, _vp, _vp, _vp,
                                       _vp, C.c_int32, C.POINTER(C.c_float), _vp]),
    "gf_sddmm": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp]),
    "gf_edge_softmax": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp]),
    "gf_spmm": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
    "gf_l2_normalize_rows": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, _vp, _vp,
                                       C.c_double, _vp]),
    "gf_l2_normalize_backward": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, _vp, _vp,
                                           _vp, C.c_double, _vp]),
    "gf_spmm_backward": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp, _vp,
                                   _vp]),
    "gf_softmax_backward": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
    "gf_sddmm_backward": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp]),
    "gf_gen_random_device": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, _vp, _vp,
                                       C.POINTER(C.c_int64), _vp]),
    "gf_gen_super_node_device": (C.c_int, [C.c_int64, C.c_double, C.c_int64, C.c_uint64, _vp, _vp,
                                           C.POINTER(C.c_int64), _vp]),
    "gf_gen_power_law_device": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_int64,
                                          _vp, _vp, C.POINTER(C.c_int64), _vp]),
    "gf_gen_molecules_device": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64,
                                          _vp, _vp, C.POINTER(C.c_int64), _vp]),
    "gf_dense_oracle_forward": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, C.POINTER(AttnDesc),
                                          C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gf_measure_metrics": (C.c_int, [C.c_void_p, C.c_void_p, _vp, C.POINTER(C.c_char_p),
                                     C.c_int32, C.POINTER(C.c_double)]),
    "gf_graph_set_split_len": (C.c_int, [_vp, C.c_int64, _vp]),
    "gf_l2_persist": (C.c_int, [C.c_size_t]),
    "gf_l2_persist_get": (C.c_int, [C.POINTER(C.c_size_t)]),
    "gf_l2_reset_persisting": (C.c_int, []),
    "gf_scratch_trim": (C.c_int, []),
    "gf_probe_scatter": (C.c_int, [C.c_int64, _vp, _vp, _vp, C.c_int32, C.c_int32,
                                   C.POINTER(C.c_float), _vp]),
    "gf_l2_policy_word": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "gf_measure_l2_gather": (C.c_int, [C.c_size_t, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                       _vp]),
    "gf_attn_bwd": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp, _vp]),
    "gf_attn_bwd_rows": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp]),
    "gf_attn_bwd_cols": (C.c_int, [_vp, C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp]),
    "gf_attn_merge_parts": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_void_p), _vp, _vp, _vp]),
    "gf_gemm_bcast": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int64, _vp, _vp,
                                C.POINTER(C.c_void_p), C.c_int32, _vp]),
    "gf_gemm_split": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int64, _vp, _vp,
                                C.POINTER(C.c_void_p), C.c_int32, _vp]),
    "gf_gemm_split": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int64, _vp, _vp,
                                C.POINTER(C.c_void_p), C.c_int32, _vp]),
    "gf_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp,
                          C.c_int32, _vp]),
    "gf_gat_logits": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp,
                                _vp, _vp]),
    "gf_gat_fanin": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp]),
}

_lib = None


class GFError(RuntimeError):
    """A GF_ERR_* status from libgraphfuse_cuda (message from gf_last_error)."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        ab_build = bool(os.environ.get("GF_CUDA_LIB"))  # A/B builds may predate newer entry points
        for name, (res, args) in SIGNATURES.items():
            if ab_build and not hasattr(L, name):
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != GF_OK:
        raise GFError(f"{what} failed (status {rc}): {lib().gf_last_error().decode()}")

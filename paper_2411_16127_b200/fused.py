"""Device-resident, multi-head entry points over the C-ABI (torch tensors in HBM).

PyTorch is plumbing here (device memory, streams); every computation is a
call into libgraphfuse_cuda.so.  Layout (see include/gf_cuda.h):
  dot (GT / AGNN): Q, K, V, O are N x (H*D); add (GAT): el, er are N x H.
"""
from __future__ import annotations

import dataclasses

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from ._capi import GF_STRAT, AttnDesc, GraphInfo, check, lib

DTYPES = {torch.float32: _capi.GF_F32, torch.float64: _capi.GF_F64}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class AttnSpec:
    """SddmmKind (dense.hpp:48-62) + multi-head shape."""

    variant: str = "dot"  # "dot" (GT/AGNN) | "add" (GAT)
    heads: int = 1
    head_dim: int = 8
    scale: float = 1.0
    slope: float = 0.2
    l2: bool = False
    # GAT layer form (GF_FLAG_LOGITS_FROM_V): Q / K are a_l / a_r (H x D, one
    # V row's layout) and el / er are computed from V's rows in the kernels
    logits_from_v: bool = False

    def desc(self, dtype) -> AttnDesc:
        if self.logits_from_v and self.variant != "add":
            raise ValueError("logits_from_v needs variant='add'")
        return AttnDesc(DTYPES[dtype], _capi.GF_ADD if self.variant == "add" else _capi.GF_DOT,
                        int(self.l2), self.heads, self.head_dim,
                        _capi.GF_FLAG_LOGITS_FROM_V if self.logits_from_v else 0,
                        float(self.scale), float(self.slope))

    @property
    def F(self) -> int:
        return self.heads * self.head_dim

    @property
    def qk_width(self) -> int:
        return self.heads if self.variant == "add" else self.F


class DeviceGraph:
    """A gf_graph_t: int32 CSR + CSC + degree-bucket schedules in HBM."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = GraphInfo()
        check(lib().gf_graph_get_info(self._h, C.byref(info)), "gf_graph_get_info")
        self.info = info
        self.n = int(info.num_nodes)
        self.e = int(info.num_edges)

    @classmethod
    def from_host_csr(cls, n, row_ptr, col, csc_ptr, csc_row, cta_threshold=0, stream=None):
        arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in (row_ptr, col, csc_ptr, csc_row)]
        h = C.c_void_p()
        check(lib().gf_graph_create(int(n), int(arrs[1].shape[0]),
                                    *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                    int(cta_threshold), _stream(stream), C.byref(h)),
              "gf_graph_create")
        return cls(h)

    @classmethod
    def from_device_csr(cls, n, row_ptr, col, csc_ptr, csc_row, cta_threshold=0, stream=None):
        ts = [t.to(torch.int32).contiguous() for t in (row_ptr, col, csc_ptr, csc_row)]
        h = C.c_void_p()
        check(lib().gf_graph_create_device(int(n), int(ts[1].numel()), *[_p(t) for t in ts],
                                           int(cta_threshold), _stream(stream), C.byref(h)),
              "gf_graph_create_device")
        return cls(h)

    @classmethod
    def from_split(cls, n, row_ptr, col, csc_ptr, csc_row, cta_threshold=0, skip_empty=False,
                   stream=None):
        """CSR and CSC with different edge sets (row-sharded graph, shard.py)."""
        rp, c, cp, cr = [t.to(torch.int32).contiguous() for t in (row_ptr, col, csc_ptr, csc_row)]
        h = C.c_void_p()
        check(lib().gf_graph_create_split(int(n), int(c.numel()), _p(rp), _p(c), int(cr.numel()),
                                          _p(cp), _p(cr), int(cta_threshold), int(skip_empty),
                                          _stream(stream), C.byref(h)), "gf_graph_create_split")
        return cls(h)

    def set_split_len(self, split_len, stream=None):
        """Edges per CTA slice of a split super row / column
        (gf_graph_set_split_len); rebuilds the CTA tables."""
        check(lib().gf_graph_set_split_len(self._h, int(split_len), _stream(stream)),
              "gf_graph_set_split_len")
        info = GraphInfo()
        check(lib().gf_graph_get_info(self._h, C.byref(info)), "gf_graph_get_info")
        self.info = info

    def schedule(self):
        """(row_order, col_order) as int32 numpy arrays (degree-descending)."""
        ro = np.zeros(max(self.n, 1), np.int32)
        co = np.zeros(max(self.n, 1), np.int32)
        check(lib().gf_graph_get_schedule(self._h, ro.ctypes.data_as(C.c_void_p),
                                          co.ctypes.data_as(C.c_void_p)), "gf_graph_get_schedule")
        return ro[: self.n], co[: self.n]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().gf_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_split_len(e, cta_threshold=0):
    """The library's default split_len for a graph of e edges (gf_cuda.h):
    max(cta_threshold or the automatic one, ceil(e / (148 * 4)))."""
    thr = cta_threshold if cta_threshold > 0 else min(16384, max(1024, e // 28416))
    return max(thr, -(-e // (148 * 4)))


def from_coo_device(n: int, src: torch.Tensor, dst: torch.Tensor, stream=None):
    """Device from_coo (graph.cpp:61-78): returns int64 (row_ptr, col, csc_ptr,
    csc_row, csc_perm) on src's device.  Raises GFError on bad ids / duplicates."""
    src = src.to(torch.int64).contiguous()
    dst = dst.to(torch.int64).contiguous()
    e = src.numel()
    dev = src.device
    rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(e, 1), dtype=torch.int64, device=dev)
    cr = torch.empty(max(e, 1), dtype=torch.int64, device=dev)
    pm = torch.empty(max(e, 1), dtype=torch.int64, device=dev)
    bad = C.c_int64(-1)
    check(lib().gf_from_coo_device(n, e, _p(src), _p(dst), _p(rp), _p(col), _p(cp), _p(cr),
                                   _p(pm), C.byref(bad), _stream(stream)), "gf_from_coo_device")
    return rp, col[:e], cp, cr[:e], pm[:e]


def attn_forward(g: DeviceGraph, spec: AttnSpec, Q, K, V, want_p=False, O=None, stats=None,
                 stream=None, strategy="smmf", workspace=None):
    """Forward; returns (O, stats) or (O, stats, P).

    strategy "smmf" (default) is the one fused launch; "pmf", "unfused" and
    "baseline" run the reference Strategy's launch structure (gf_cuda.h
    GF_STRAT_*).  stats is N x H x 4 softmax records {m, log2 l, aux, delta}
    (gf_cuda.h).  workspace: optional preallocated scratch (strategy_workspace)."""
    n = g.n
    dt = V.dtype
    if O is None:
        O = torch.empty(n, spec.F, dtype=dt, device=V.device)
    if stats is None:
        stats = torch.empty(n, spec.heads, 4, dtype=dt, device=V.device)
    P = torch.empty(max(g.e, 1), spec.heads, dtype=dt, device=V.device) if want_p else None
    d = spec.desc(dt)
    if strategy == "smmf" and workspace is None:
        check(lib().gf_attn_fwd(g.handle, C.byref(d), _p(Q), _p(K), _p(V), _p(O), _p(stats),
                                _p(P), _stream(stream)), "gf_attn_fwd")
    else:
        ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        check(lib().gf_attn_fwd_strategy(g.handle, C.byref(d), GF_STRAT[strategy], _p(Q), _p(K),
                                         _p(V), _p(O), _p(stats), _p(P), _p(workspace), ws_bytes,
                                         _stream(stream)), "gf_attn_fwd_strategy")
    return (O, stats, P[: g.e]) if want_p else (O, stats)


def strategy_workspace(g: DeviceGraph, spec: AttnSpec, strategy: str, dtype=torch.float32,
                       device="cuda", want_p=False):
    """Scratch buffer for attn_forward(strategy=...) (None when none is needed)."""
    n = C.c_size_t()
    check(lib().gf_attn_fwd_workspace(g.handle, C.byref(spec.desc(dtype)), GF_STRAT[strategy],
                                      int(want_p), C.byref(n)), "gf_attn_fwd_workspace")
    return torch.empty(n.value, dtype=torch.uint8, device=device) if n.value else None


def lse_of(stats):
    """log-sum-exp per (row, head) from the records: m + log2(l) * ln 2."""
    return stats[..., 0] + stats[..., 1] * 0.6931471805599453


def attn_backward(g: DeviceGraph, spec: AttnSpec, Q, K, V, O, stats, dO, dQ=None, dK=None,
                  dV=None, stream=None):
    """Pass A (CSR) + pass B (CSC); returns (dQ|del, dK|der, dV)."""
    dt = V.dtype
    dev = V.device
    if dQ is None:
        dQ = torch.empty(g.n, spec.qk_width, dtype=dt, device=dev)
    if dK is None:
        dK = torch.empty(g.n, spec.qk_width, dtype=dt, device=dev)
    if dV is None:
        dV = torch.empty(g.n, spec.F, dtype=dt, device=dev)
    d = spec.desc(dt)
    check(lib().gf_attn_bwd(g.handle, C.byref(d), _p(Q), _p(K), _p(V), _p(O), _p(stats), _p(dO),
                            _p(dQ), _p(dK), _p(dV), _stream(stream)), "gf_attn_bwd")
    return dQ, dK, dV


def attn_backward_rows(g, spec, Q, K, V, O, stats, dO, dK, stream=None):
    """Pass A only: dK | der, and delta into the stats records (CSR rows)."""
    d = spec.desc(V.dtype)
    check(lib().gf_attn_bwd_rows(g.handle, C.byref(d), _p(Q), _p(K), _p(V), _p(O), _p(stats),
                                 _p(dO), _p(dK), _stream(stream)), "gf_attn_bwd_rows")


def attn_backward_cols(g, spec, Q, K, V, stats, dO, dQ, dV, stream=None):
    """Pass B only: dQ | del and dV (CSC columns), reading pass A's records."""
    d = spec.desc(V.dtype)
    check(lib().gf_attn_bwd_cols(g.handle, C.byref(d), _p(Q), _p(K), _p(V), _p(stats), _p(dO),
                                 _p(dQ), _p(dV), _stream(stream)), "gf_attn_bwd_cols")


class FusedAttention(torch.autograd.Function):
    """torch.autograd wrapper: forward saves only (O, stats); backward recomputes."""

    @staticmethod
    def forward(ctx, g, spec, Q, K, V):
        Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
        O, stats = attn_forward(g, spec, Q, K, V)
        ctx.g, ctx.spec = g, spec
        ctx.save_for_backward(Q, K, V, O, stats)
        return O

    @staticmethod
    def backward(ctx, dO):
        Q, K, V, O, stats = ctx.saved_tensors
        dQ, dK, dV = attn_backward(ctx.g, ctx.spec, Q, K, V, O, stats, dO.contiguous())
        return None, None, dQ, dK, dV


def gemm(A, B, trans_a=False, out=None, accumulate=False, stream=None):
    """C = A @ B or A^T @ B (gf_gemm, row-major)."""
    if trans_a:
        K, M = A.shape
    else:
        M, K = A.shape
    N = B.shape[1]
    if out is None:
        out = torch.empty(M, N, dtype=A.dtype, device=A.device)
    check(lib().gf_gemm(DTYPES[A.dtype], int(trans_a), M, N, K, _p(A), _p(B), _p(out),
                        int(accumulate), _stream(stream)), "gf_gemm")
    return out


def attn_merge_parts(spec: AttnSpec, row_ptrs, O_parts, rec_parts, O, stats, stream=None):
    """Combine source-phased forward partials (gf_attn_merge_parts): part k =
    the forward over the in-edges from source block k (row pointer row_ptrs[k],
    normalised O_parts[k], records rec_parts[k]); all row-relative views of the
    same rows.  Writes O and the records' {m, log2 l, aux}."""
    n = len(O_parts)
    if not (len(row_ptrs) == len(rec_parts) == n):
        raise ValueError("attn_merge_parts: one row pointer, O and record table per part")
    rows = O.shape[0]
    arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() for t in ts])  # noqa: E731
    check(lib().gf_attn_merge_parts(DTYPES[O.dtype], rows, spec.heads, spec.head_dim, n,
                                    arr(row_ptrs), arr(O_parts), arr(rec_parts), _p(O), _p(stats),
                                    _stream(stream)), "gf_attn_merge_parts")
    return O, stats


def gemm_bcast(A, B, outs, stream=None):
    """C = A @ B stored tile by tile into every tensor of `outs` (gf_gemm_bcast):
    outs[0] local, outs[1..] the same rows of peer ranks' tables (peer-mapped
    views, e.g. torch symmetric memory buffers).  fp32, N % 32 == 0."""
    M, K = A.shape
    N = B.shape[1]
    for o in outs:
        if tuple(o.shape) != (M, N) or not o.is_contiguous():
            raise ValueError("gemm_bcast: every destination must be a contiguous M x N view")
    arr = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    check(lib().gf_gemm_bcast(DTYPES[A.dtype], M, N, K, _p(A), _p(B), arr, len(outs),
                              _stream(stream)), "gf_gemm_bcast")
    return outs[0]


def gemm_split(A, B, outs, stream=None):
    """C = A @ B with column block j of C written to outs[j] (gf_gemm_split):
    X @ [W_q | W_k | W_v] -> Q, K, V in one tcgen05 GEMM.  fp32, each block
    a multiple of 32 columns."""
    M, K = A.shape
    N = B.shape[1]
    w = N // max(1, len(outs))
    for o in outs:
        if tuple(o.shape) != (M, w) or not o.is_contiguous():
            raise ValueError("gemm_split: every destination must be a contiguous M x N/len(outs) view")
    arr = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    check(lib().gf_gemm_split(DTYPES[A.dtype], M, N, K, _p(A), _p(B), arr, len(outs),
                              _stream(stream)), "gf_gemm_split")
    return outs


def gemm_split(A, B, outs, stream=None):
    """C = A @ B with column block j of C written to outs[j] (gf_gemm_split):
    X @ [W_q | W_k | W_v] -> Q, K, V in one tcgen05 GEMM.  fp32, each block
    a multiple of 32 columns."""
    M, K = A.shape
    N = B.shape[1]
    w = N // max(1, len(outs))
    for o in outs:
        if tuple(o.shape) != (M, w) or not o.is_contiguous():
            raise ValueError("gemm_split: every destination must be a contiguous M x N/len(outs) view")
    arr = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    check(lib().gf_gemm_split(DTYPES[A.dtype], M, N, K, _p(A), _p(B), arr, len(outs),
                              _stream(stream)), "gf_gemm_split")
    return outs


def gat_logits(Hf, a_l, a_r, heads, head_dim, stream=None, el=None, er=None):
    n = Hf.shape[0]
    el = torch.empty(n, heads, dtype=Hf.dtype, device=Hf.device) if el is None else el
    er = torch.empty_like(el) if er is None else er
    check(lib().gf_gat_logits(DTYPES[Hf.dtype], n, heads, head_dim, _p(Hf), _p(a_l), _p(a_r),
                              _p(el), _p(er), _stream(stream)), "gf_gat_logits")
    return el, er


def gat_fanin(Hf, a_l, a_r, dV, d_el, d_er, heads, head_dim, stream=None):
    n = Hf.shape[0]
    dH = torch.empty_like(dV)
    dal = torch.empty(heads * head_dim, dtype=Hf.dtype, device=Hf.device)
    dar = torch.empty_like(dal)
    check(lib().gf_gat_fanin(DTYPES[Hf.dtype], n, heads, head_dim, _p(Hf), _p(a_l), _p(a_r),
                             _p(dV), _p(d_el), _p(d_er), _p(dH), _p(dal), _p(dar),
                             _stream(stream)), "gf_gat_fanin")
    return dH, dal, dar


# ---- single-step operators (the unfused schedule; gf_cuda.h "single-step") --
def _edge_buf(g, heads, dt, dev):
    return torch.empty(max(g.e, 1), heads, dtype=dt, device=dev)


def sddmm(g: DeviceGraph, spec: AttnSpec, Q, K, S=None, stream=None):
    """S[E x H] (kernels.hpp:106-117)."""
    S = _edge_buf(g, spec.heads, Q.dtype, Q.device) if S is None else S
    check(lib().gf_sddmm(g.handle, C.byref(spec.desc(Q.dtype)), _p(Q), _p(K), _p(S),
                         _stream(stream)), "gf_sddmm")
    return S[: g.e]


def edge_softmax(g: DeviceGraph, heads, S, P=None, stream=None):
    """P[E x H] (kernels.hpp:65-82)."""
    P = _edge_buf(g, heads, S.dtype, S.device) if P is None else P
    check(lib().gf_edge_softmax(g.handle, DTYPES[S.dtype], heads, _p(S), _p(P), _stream(stream)),
          "gf_edge_softmax")
    return P[: g.e]


def spmm(g: DeviceGraph, heads, head_dim, P, V, O=None, stream=None):
    """O = P V per head (kernels.hpp:85-102)."""
    O = torch.empty(g.n, heads * head_dim, dtype=V.dtype, device=V.device) if O is None else O
    check(lib().gf_spmm(g.handle, DTYPES[V.dtype], heads, head_dim, _p(P), _p(V), _p(O),
                        _stream(stream)), "gf_spmm")
    return O


def l2_normalize_rows(X, heads, head_dim, eps=1e-12, stream=None):
    Y = torch.empty_like(X)
    check(lib().gf_l2_normalize_rows(DTYPES[X.dtype], X.shape[0], heads, head_dim, _p(X), _p(Y),
                                     eps, _stream(stream)), "gf_l2_normalize_rows")
    return Y


def l2_normalize_backward(X, dY, heads, head_dim, eps=1e-12, stream=None):
    dX = torch.empty_like(X)
    check(lib().gf_l2_normalize_backward(DTYPES[X.dtype], X.shape[0], heads, head_dim, _p(X),
                                         _p(dY), _p(dX), eps, _stream(stream)),
          "gf_l2_normalize_backward")
    return dX


def spmm_backward(g: DeviceGraph, heads, head_dim, P, V, dO, stream=None):
    """(dP, dV) (autograd.hpp:33-58)."""
    dP = _edge_buf(g, heads, V.dtype, V.device)
    dV = torch.empty_like(V)
    check(lib().gf_spmm_backward(g.handle, DTYPES[V.dtype], heads, head_dim, _p(P), _p(V), _p(dO),
                                 _p(dP), _p(dV), _stream(stream)), "gf_spmm_backward")
    return dP[: g.e], dV


def softmax_backward(g: DeviceGraph, heads, P, dP, stream=None):
    """dS (autograd.hpp:62-73)."""
    dS = _edge_buf(g, heads, P.dtype, P.device)
    check(lib().gf_softmax_backward(g.handle, DTYPES[P.dtype], heads, _p(P), _p(dP), _p(dS),
                                    _stream(stream)), "gf_softmax_backward")
    return dS[: g.e]


def sddmm_backward(g: DeviceGraph, spec: AttnSpec, Q, K, dS, stream=None):
    """(dQ|del, dK|der) (autograd.hpp:102-154)."""
    dQ = torch.empty(g.n, spec.qk_width, dtype=Q.dtype, device=Q.device)
    dK = torch.empty_like(dQ)
    check(lib().gf_sddmm_backward(g.handle, C.byref(spec.desc(Q.dtype)), _p(Q), _p(K), _p(dS),
                                  _p(dQ), _p(dK), _stream(stream)), "gf_sddmm_backward")
    return dQ, dK


def attn_backward_unfused(g: DeviceGraph, spec: AttnSpec, Q, K, V, P, dO, stream=None):
    """The reference's unfused backward (autograd.hpp:158-170, 196-203): dP/dV,
    then dS, then dQ/dK, with the E x H edge gradients in HBM.  Returns
    (dQ|del, dK|der, dV, dP, dS)."""
    if spec.logits_from_v:  # the single-step ops take explicit el / er tables
        Q, K = gat_logits(V, Q, K, spec.heads, spec.head_dim, stream=stream)
        spec = dataclasses.replace(spec, logits_from_v=False)
    dP, dV = spmm_backward(g, spec.heads, spec.head_dim, P, V, dO, stream=stream)
    dS = softmax_backward(g, spec.heads, P, dP, stream=stream)
    dQ, dK = sddmm_backward(g, spec, Q, K, dS, stream=stream)
    return dQ, dK, dV, dP, dS


# ---- synthetic graphs on the device (gf_cuda.h "synthetic graphs") ---------
def gen_random_device(n, avg_degree, seed=0, device="cuda", stream=None):
    """(src, dst) int64 device COO: exactly round(n*avg) distinct uniform edges."""
    e = int(avg_degree * n + 0.5)
    src = torch.empty(max(e, 1), dtype=torch.int64, device=device)
    dst = torch.empty_like(src)
    out = C.c_int64()
    check(lib().gf_gen_random_device(n, float(avg_degree), seed, _p(src), _p(dst), C.byref(out),
                                     _stream(stream)), "gf_gen_random_device")
    return src[: out.value], dst[: out.value]


def gen_super_node_device(n, avg_degree, hub_degree, seed=0, device="cuda", stream=None):
    """(src, dst): node 0 with exactly hub_degree in-neighbours + uniform edges."""
    e = max(hub_degree, int(avg_degree * n + 0.5))
    src = torch.empty(max(e, 1), dtype=torch.int64, device=device)
    dst = torch.empty_like(src)
    out = C.c_int64()
    check(lib().gf_gen_super_node_device(n, float(avg_degree), hub_degree, seed, _p(src), _p(dst),
                                         C.byref(out), _stream(stream)),
          "gf_gen_super_node_device")
    return src[: out.value], dst[: out.value]


def gen_power_law_device(n, max_degree, exponent, seed=0, device="cuda", stream=None):
    """(src, dst): in-degree sequence round(max (r+1)^-exponent) on hashed ids."""
    cap = int(np.rint(max_degree * (np.arange(n, dtype=np.float64) + 1.0) ** -exponent).sum())
    src = torch.empty(max(cap, 1), dtype=torch.int64, device=device)
    dst = torch.empty_like(src)
    out = C.c_int64()
    check(lib().gf_gen_power_law_device(n, max_degree, float(exponent), seed, cap, _p(src),
                                        _p(dst), C.byref(out), _stream(stream)),
          "gf_gen_power_law_device")
    return src[: out.value], dst[: out.value]


def gen_molecules_device(mols, atoms, rings, seed=0, device="cuda", stream=None):
    """(src, dst): `mols` disjoint molecules of `atoms` ids (batch_graphs
    layout), each a spanning tree + `rings` bonds, both directions, deduped."""
    cap = 2 * mols * (atoms - 1 + rings)
    src = torch.empty(max(cap, 1), dtype=torch.int64, device=device)
    dst = torch.empty_like(src)
    out = C.c_int64()
    check(lib().gf_gen_molecules_device(mols, atoms, rings, seed, cap, _p(src), _p(dst),
                                        C.byref(out), _stream(stream)), "gf_gen_molecules_device")
    return src[: out.value], dst[: out.value]


_REGION_FN = C.CFUNCTYPE(None, C.c_void_p)


def measure_metrics(fn, metrics, prep=None):
    """Hardware counters of the kernels `fn()` launches (gf_measure_metrics:
    CUPTI range profiler, one range, user replay; `prep()` runs before every
    pass outside the range, e.g. an L2 flush).  Returns {metric: value}.
    Raises GFError (status GF_ERR_UNSUPPORTED = 4) without CUPTI / permission."""
    cb = _REGION_FN(lambda _u: fn())
    pcb = _REGION_FN(lambda _u: prep()) if prep is not None else None
    names = (C.c_char_p * len(metrics))(*[m.encode() for m in metrics])
    vals = (C.c_double * len(metrics))()
    check(lib().gf_measure_metrics(C.cast(pcb, C.c_void_p) if pcb else None, C.cast(cb, C.c_void_p),
                                   None, names, len(metrics), vals), "gf_measure_metrics")
    return {m: float(v) for m, v in zip(metrics, vals)}


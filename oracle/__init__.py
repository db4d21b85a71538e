"""TEST INFRASTRUCTURE ONLY — CPU checkers for the B200 fused AT-GNN path.

Two libraries, both loaded through ctypes:

* ``oracle/_build/libgforacle.so`` — this repo's plain-C restatement of the
  reference algorithm (``gf_oracle.c``; every function cites the reference
  file:line it restates).
* ``oracle/_ref/libgfref.so`` — the UNMODIFIED reference (``graphfuse``),
  compiled from its own sources under /root/reference by ``oracle/Makefile``.
  It travels to the GPU box prebuilt; the sources do not.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product path (``paper_2411_16127_b200``)
never does, and fails loudly when its CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libgforacle.so")
REF_SO = os.path.join(HERE, "_ref", "libgfref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def build() -> None:
    """Compile the restatement (and, where the reference exists, _ref)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


_ora = None
_ref = None


def lib():
    global _ora
    if _ora is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _ora = C.CDLL(ORACLE_SO)
        _ora.gfo_from_coo.restype = C.c_int
        _ora.gfo_from_coo.argtypes = [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        _ora.gfo_schedule.restype = None
        _ora.gfo_schedule.argtypes = [C.c_int64, _vp, C.c_int64, _vp, _vp, _vp, _vp]
        for sfx in ("f32", "f64"):
            f = getattr(_ora, "gfo_forward_" + sfx)
            f.restype = C.c_int
            f.argtypes = [C.c_int64, C.c_int64, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int,
                          C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp]
            b = getattr(_ora, "gfo_backward_" + sfx)
            b.restype = C.c_int
            b.argtypes = [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int,
                          C.c_int, C.c_int, C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp,
                          _vp, _vp]
            b2 = getattr(_ora, "gfo_backward2_" + sfx)
            b2.restype = C.c_int
            b2.argtypes = b.argtypes + [_vp, _vp]
    return _ora


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference itself (compiled from /root/reference sources)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        _ref = C.CDLL(REF_SO)
        _ref.gfref_last_error.restype = C.c_char_p
        for name in ("gfref_from_coo",):
            getattr(_ref, name).restype = _vp
            getattr(_ref, name).argtypes = [C.c_int64, C.c_int64, _vp, _vp]
        _ref.gfref_graph_adopt.restype = _vp
        _ref.gfref_graph_adopt.argtypes = [C.c_int64, C.c_int64] + [_vp] * 5
        _ref.gfref_gen_random.restype = _vp
        _ref.gfref_gen_random.argtypes = [C.c_int64, C.c_double, C.c_uint64]
        _ref.gfref_gen_super_node.restype = _vp
        _ref.gfref_gen_super_node.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_uint64]
        _ref.gfref_graph_free.argtypes = [_vp]
        _ref.gfref_num_nodes.restype = C.c_int64
        _ref.gfref_num_nodes.argtypes = [_vp]
        _ref.gfref_num_edges.restype = C.c_int64
        _ref.gfref_num_edges.argtypes = [_vp]
        _ref.gfref_graph_arrays.argtypes = [_vp] * 6
        for sfx in ("f32", "f64"):
            f = getattr(_ref, "gfref_forward_" + sfx)
            f.restype = C.c_int
            f.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                          C.c_int, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]
            b = getattr(_ref, "gfref_backward_" + sfx)
            b.restype = C.c_int
            b.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                          C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        _ref.gfref_time_head_f32.restype = C.c_int
        _ref.gfref_time_head_f32.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double,
                                             C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        _ref.gfref_time_step_f32.restype = C.c_int
        _ref.gfref_time_step_f32.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_double, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        _ref.gfref_time_conv_f32.restype = C.c_int
        _ref.gfref_time_conv_f32.argtypes = [_vp, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                             C.c_double, C.c_double] + [_vp] * 8
        _ref.gfref_forward_counters.restype = C.c_int
        _ref.gfref_forward_counters.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                                C.c_int64, C.c_int, _vp, _vp, C.c_int64, _vp]
        _ref.gfref_conv_f64.restype = C.c_int
        _ref.gfref_conv_f64.argtypes = [_vp, C.c_int, C.c_int64, C.c_int64, C.c_double,
                                        C.c_double] + [_vp] * 13
        _ref.gfref_gradcheck.restype = C.c_double
        _ref.gfref_gradcheck.argtypes = [_vp, C.c_int, C.c_int64, C.c_uint64, C.c_double]
        _ref.gfref_random_matrix_f64.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                                 C.c_double, _vp]
        _ref.gfref_random_matrix_f32.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_float,
                                                 C.c_float, _vp]
    return _ref


# ------------------------------------------------------------------ graphs --
class CSR:
    """Canonical hybrid topology in the reference layout (graph.hpp:24-38)."""

    def __init__(self, n, row_ptr, col, csc_ptr, csc_row, csc_perm):
        self.n = int(n)
        self.e = int(col.shape[0])
        self.row_ptr, self.col = row_ptr, col
        self.csc_ptr, self.csc_row, self.csc_perm = csc_ptr, csc_row, csc_perm

    @property
    def coo_dst(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))


class OracleError(RuntimeError):
    pass


def from_coo(n, src, dst) -> CSR:
    """gf_oracle restatement of graph.cpp:61-78."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    e = src.shape[0]
    rp = np.zeros(n + 1, np.int64)
    col = np.zeros(max(e, 1), np.int64)
    cp = np.zeros(n + 1, np.int64)
    cr = np.zeros(max(e, 1), np.int64)
    perm = np.zeros(max(e, 1), np.int64)
    bad = np.zeros(1, np.int64)
    rc = lib().gfo_from_coo(n, e, _ptr(src), _ptr(dst), _ptr(rp), _ptr(col), _ptr(cp), _ptr(cr),
                            _ptr(perm), _ptr(bad))
    if rc == 1:
        raise OracleError(f"from_coo: node id out of range at input edge {bad[0]}")
    if rc == 2:
        raise OracleError(f"from_coo: duplicate edge at sorted position {bad[0]}")
    return CSR(n, rp, col[:e], cp, cr[:e], perm[:e])


def schedule(n, ptr, cta_threshold, want_small=False):
    order = np.zeros(max(n, 1), np.int32)
    nc = np.zeros(1, np.int64)
    nz = np.zeros(1, np.int64)
    ns = np.zeros(1, np.int64)
    lib().gfo_schedule(n, _ptr(np.ascontiguousarray(ptr, np.int64)), cta_threshold, _ptr(order),
                       _ptr(nc), _ptr(nz), _ptr(ns))
    if want_small:
        return order[:n], int(nc[0]), int(nz[0]), int(ns[0])
    return order[:n], int(nc[0]), int(nz[0])


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def forward(g: CSR, Q, K, V, H, D, variant="dot", l2=False, scale=1.0, slope=0.2,
            want_p=False, want_lse=False):
    """Multi-head forward restatement (engine.hpp:192-231 per head)."""
    dt = V.dtype
    var = 1 if variant == "add" else 0
    O = np.zeros((g.n, H * D), dt)
    P = np.zeros((g.e, H), dt) if want_p else None
    lse = np.zeros((g.n, H), dt) if want_lse else None
    f = getattr(lib(), "gfo_forward_" + _sfx(dt))
    f(g.n, g.e, _ptr(g.row_ptr), _ptr(g.col), H, D, var, int(l2), scale, slope,
      _ptr(np.ascontiguousarray(Q, dt)), _ptr(np.ascontiguousarray(K, dt)),
      _ptr(np.ascontiguousarray(V, dt)), _ptr(O), _ptr(P), _ptr(lse))
    out = [O]
    if want_p:
        out.append(P)
    if want_lse:
        out.append(lse)
    return out[0] if len(out) == 1 else tuple(out)


def backward(g: CSR, Q, K, V, dO, H, D, variant="dot", l2=False, scale=1.0, slope=0.2,
             want_edge_grads=False):
    """Multi-head backward restatement (autograd.hpp:158-170 per head).
    Returns (dQ, dK, dV), plus (dP, dS) (E x H, CSR order) on request."""
    dt = V.dtype
    var = 1 if variant == "add" else 0
    w = H if var == 1 else H * D
    dQ = np.zeros((g.n, w), dt)
    dK = np.zeros((g.n, w), dt)
    dV = np.zeros((g.n, H * D), dt)
    dP = np.zeros((max(g.e, 1), H), dt) if want_edge_grads else None
    dS = np.zeros((max(g.e, 1), H), dt) if want_edge_grads else None
    f = getattr(lib(), "gfo_backward2_" + _sfx(dt))
    f(g.n, g.e, _ptr(g.row_ptr), _ptr(g.col), _ptr(g.csc_ptr), _ptr(g.csc_row), _ptr(g.csc_perm),
      H, D, var, int(l2), scale, slope, _ptr(np.ascontiguousarray(Q, dt)),
      _ptr(np.ascontiguousarray(K, dt)), _ptr(np.ascontiguousarray(V, dt)),
      _ptr(np.ascontiguousarray(dO, dt)), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dP), _ptr(dS))
    if want_edge_grads:
        return dQ, dK, dV, dP[: g.e], dS[: g.e]
    return dQ, dK, dV


# --------------------------------------------------------------- reference --
class RefGraph:
    """Owning handle to a reference ``graphfuse::Graph``."""

    def __init__(self, handle):
        if not handle:
            raise OracleError(ref().gfref_last_error().decode())
        self.h = handle
        self.n = ref().gfref_num_nodes(handle)
        self.e = ref().gfref_num_edges(handle)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.gfref_graph_free(self.h)
            self.h = None

    def arrays(self) -> CSR:
        n, e = self.n, self.e
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(max(e, 1), np.int64)
        cp = np.zeros(n + 1, np.int64)
        cr = np.zeros(max(e, 1), np.int64)
        pm = np.zeros(max(e, 1), np.int64)
        ref().gfref_graph_arrays(self.h, _ptr(rp), _ptr(col), _ptr(cp), _ptr(cr), _ptr(pm))
        return CSR(n, rp, col[:e], cp, cr[:e], pm[:e])


def ref_from_coo(n, src, dst) -> RefGraph:
    src = np.ascontiguousarray(src, np.int64)
    dst = np.ascontiguousarray(dst, np.int64)
    return RefGraph(ref().gfref_from_coo(n, src.shape[0], _ptr(src), _ptr(dst)))


def ref_adopt(g: CSR) -> RefGraph:
    return RefGraph(ref().gfref_graph_adopt(g.n, g.e, _ptr(g.row_ptr), _ptr(g.col),
                                            _ptr(g.csc_ptr), _ptr(g.csc_row),
                                            _ptr(g.csc_perm)))


def ref_gen_random(n, avg, seed) -> RefGraph:
    return RefGraph(ref().gfref_gen_random(n, avg, seed))


def ref_gen_super_node(n, avg, hub, seed) -> RefGraph:
    return RefGraph(ref().gfref_gen_super_node(n, avg, hub, seed))


STRATEGIES = {"smmf": 0, "pmf": 1, "unfused": 2, "baseline": 3}


def ref_forward(g: RefGraph, Q, K, V, H, D, variant="dot", l2=False, scale=1.0, slope=0.2,
                strategy="smmf", budget=1 << 30, want_p=False):
    dt = V.dtype
    O = np.zeros((g.n, H * D), dt)
    P = np.zeros((g.e, H), dt) if want_p else None
    f = getattr(ref(), "gfref_forward_" + _sfx(dt))
    rc = f(g.h, H, D, 1 if variant == "add" else 0, scale, slope, int(l2), STRATEGIES[strategy],
           budget, _ptr(np.ascontiguousarray(Q, dt)), _ptr(np.ascontiguousarray(K, dt)),
           _ptr(np.ascontiguousarray(V, dt)), _ptr(O), _ptr(P), None)
    if rc:
        raise OracleError(ref().gfref_last_error().decode())
    return (O, P) if want_p else O


def ref_backward(g: RefGraph, Q, K, V, dO, H, D, variant="dot", l2=False, scale=1.0, slope=0.2,
                 fused=True):
    dt = V.dtype
    var = 1 if variant == "add" else 0
    w = H if var == 1 else H * D
    dQ = np.zeros((g.n, w), dt)
    dK = np.zeros((g.n, w), dt)
    dV = np.zeros((g.n, H * D), dt)
    f = getattr(ref(), "gfref_backward_" + _sfx(dt))
    rc = f(g.h, H, D, var, scale, slope, int(l2), int(fused), _ptr(np.ascontiguousarray(Q, dt)),
           _ptr(np.ascontiguousarray(K, dt)), _ptr(np.ascontiguousarray(V, dt)),
           _ptr(np.ascontiguousarray(dO, dt)), _ptr(dQ), _ptr(dK), _ptr(dV), None)
    if rc:
        raise OracleError(ref().gfref_last_error().decode())
    return dQ, dK, dV


def ref_random_matrix(rows, cols, seed, lo=-1.0, hi=1.0, dtype=np.float64):
    out = np.zeros((rows, cols), dtype)
    if np.dtype(dtype) == np.float64:
        ref().gfref_random_matrix_f64(rows, cols, seed, lo, hi, _ptr(out))
    else:
        ref().gfref_random_matrix_f32(rows, cols, seed, lo, hi, _ptr(out))
    return out


def rel_err(a, b) -> float:
    """The reference's parity metric |a-b| / max(|a|,|b|,1) (bench.cpp:106-115)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))

"""GPU, BASELINE full sizes: the C4 Reddit-shape (114 M edges, hub in-degree
~20.6 k) GAT 8x8 and the C5 ogbn-products-shape (62 M edges) GT 8x16 layers,
checked through size-independent properties (the oracle cannot run the whole
graph in a test) plus oracle parity on sampled rows:

* normalisation: with V = 1 every non-empty row's output is exactly the
  softmax mass, 1 (empty rows: 0);
* sampled rows (incl. the largest hub) == the CPU oracle run on those rows'
  complete in-edge sets with the full node tables (forward O and pass A's
  dK|der, the destination-owned gradients);
* transposed aggregation (pass B): sum_u dV[u] = sum over non-empty rows v of
  dO[v] (each row's probabilities sum to 1), and for GAT sum_u del[u] =
  sum_v der[v] (both are sum_e dS_e lrelu'(pre_e));
* sampled COLUMNS (incl. the largest out-hub) == the oracle on the complete
  in-edge sets of every destination they reach, so pass B's source-owned
  gradients dV and dQ|del are checked elementwise (autograd.hpp:33-58,
  120-154: dV and dQ over CSC);
* linearity in dO: gradients of 2 dO are exactly 2x (power-of-two scaling);
* determinism: a repeated step is bitwise identical.
Tolerance for fp32 sums over 10^8 terms: relative 1e-4 of the summed
magnitude (sum of |terms|)."""
import numpy as np
import pytest

import oracle
from oracle import rel_err

pytestmark = pytest.mark.gpu

SHAPES = {
    "c4": ("reddit", "add", 8, 8),
    "c5gat": ("products", "add", 8, 8),
    "c5gt": ("products", "dot", 8, 16),
}


def _setup(name):
    import os
    import sys

    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2411_16127_b200 import fused

    graph, variant, H, D = SHAPES[name]
    dev = torch.device("cuda")
    n, src, dst = bench.gen_graph_device(graph, dev, seed=5)
    rp, col, cp, cr, _ = fused.from_coo_device(n, src, dst)
    del src, dst
    dg = fused.DeviceGraph.from_device_csr(n, rp, col, cp, cr)
    spec = fused.AttnSpec(variant, H, D, scale=(1.0 / np.sqrt(D)) if variant == "dot" else 1.0,
                          slope=0.2)
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    qk = spec.qk_width
    amp = 2.0 if variant == "add" else 1.0
    u = lambda *s, a=1.0: (torch.rand(*s, device=dev, generator=g) * 2 - 1) * a  # noqa: E731
    Q, K, V, dO = u(n, qk, a=amp), u(n, qk, a=amp), u(n, H * D), u(n, H * D)
    return n, rp, col, dg, spec, Q, K, V, dO


def _sub_rows(n, rp_h, col_h, rows):
    """oracle.CSR of the complete in-edge sets of `rows` (other rows empty)."""
    segs = [col_h[rp_h[v]: rp_h[v + 1]] for v in rows]
    counts = np.zeros(n, np.int64)
    counts[rows] = [len(s) for s in segs]
    sub_ptr = np.zeros(n + 1, np.int64)
    sub_ptr[1:] = np.cumsum(counts)
    sub_col = np.concatenate(segs) if segs else np.zeros(0, np.int64)
    dst = np.repeat(rows, [len(s) for s in segs])
    order = np.argsort(sub_col, kind="stable")
    csc_ptr = np.zeros(n + 1, np.int64)
    csc_ptr[1:] = np.cumsum(np.bincount(sub_col, minlength=n))
    return oracle.CSR(n, sub_ptr, sub_col, csc_ptr, dst[order], order.astype(np.int64))


def _step(dg, spec, Q, K, V, dO):
    from paper_2411_16127_b200 import fused

    O, st = fused.attn_forward(dg, spec, Q, K, V)
    dQ, dK, dV = fused.attn_backward(dg, spec, Q, K, V, O, st, dO)
    return O, st, dQ, dK, dV


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_fullsize_properties(cuda, name):
    import torch

    from paper_2411_16127_b200 import fused

    n, rp, col, dg, spec, Q, K, V, dO = _setup(name)
    H, D = spec.heads, spec.head_dim
    deg = (rp[1:] - rp[:-1]).to(torch.int64)
    nonempty = deg > 0

    # normalisation: V = 1 -> O = 1 on non-empty rows, 0 on empty rows
    O1, _ = fused.attn_forward(dg, spec, Q, K, torch.ones_like(V))
    assert float((O1[nonempty] - 1).abs().max()) < 1e-5
    if bool((~nonempty).any()):
        assert float(O1[~nonempty].abs().max()) == 0.0
    del O1

    O, st, dQ, dK, dV = _step(dg, spec, Q, K, V, dO)
    torch.cuda.synchronize()

    # transposed aggregation: sum_u dV[u] == sum_{non-empty v} dO[v]
    lhs = dV.double().sum(0)
    rhs = dO[nonempty].double().sum(0)
    mag = dV.double().abs().sum(0) + dO.double().abs().sum(0)
    assert float(((lhs - rhs).abs() / mag).max()) < 1e-4
    if spec.variant == "add":  # sum del == sum der (both sum_e dS_e lrelu'(pre_e))
        a, b = dQ.double().sum(0), dK.double().sum(0)
        m = dQ.double().abs().sum(0) + dK.double().abs().sum(0)
        assert float(((a - b).abs() / m).max()) < 1e-4

    # linearity in dO (power-of-two scaling is exact) and determinism
    O2, st2, dQ2, dK2, dV2 = _step(dg, spec, Q, K, V, 2 * dO)
    assert torch.equal(dV2, 2 * dV) and torch.equal(dQ2, 2 * dQ) and torch.equal(dK2, 2 * dK)
    O3, st3, dQ3, dK3, dV3 = _step(dg, spec, Q, K, V, dO)
    assert torch.equal(O3, O) and torch.equal(dV3, dV) and torch.equal(dQ3, dQ) and torch.equal(dK3, dK)

    # sampled rows vs the oracle on their complete in-edge sets
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[int(torch.argmax(deg))],
                                     rng.choice(n, 300, replace=False)]))
    rp_h, col_h = rp.cpu().numpy().astype(np.int64), col.cpu().numpy().astype(np.int64)
    sub = _sub_rows(n, rp_h, col_h, rows)
    hQ, hK, hV, hdO = (x.cpu().numpy() for x in (Q, K, V, dO))
    O_ref = oracle.forward(sub, hQ, hK, hV, H, D, spec.variant, False, spec.scale, 0.2)
    _, dK_ref, _ = oracle.backward(sub, hQ, hK, hV, hdO, H, D, spec.variant, False, spec.scale, 0.2)
    got_O, got_dK = O.cpu().numpy()[rows], dK.cpu().numpy()[rows]
    assert rel_err(got_O, O_ref[rows]) <= 1e-4
    assert rel_err(got_dK, dK_ref[rows]) <= 1e-4
    del sub, O_ref, dK_ref

    # sampled columns (pass B, source-owned): every out-edge u -> v of a
    # sampled u lands in a complete row v of the sub-graph, so the oracle's
    # dV[u] and dQ|del[u] there equal the full graph's
    out_deg = np.bincount(col_h, minlength=n)
    k = 40 if name == "c4" else 300  # C4 rows reached are hub-heavy (~670 in-edges each)
    cols = np.unique(np.concatenate([[int(np.argmax(out_deg))],
                                     rng.choice(n, k, replace=False)]))
    is_col = np.zeros(n, bool)
    is_col[cols] = True
    dst_all = np.repeat(np.arange(n), np.diff(rp_h))
    reach = np.unique(dst_all[is_col[col_h]])
    del dst_all
    sub = _sub_rows(n, rp_h, col_h, reach)
    dQ_ref, _, dV_ref = oracle.backward(sub, hQ, hK, hV, hdO, H, D, spec.variant, False,
                                        spec.scale, 0.2)
    assert rel_err(dV.cpu().numpy()[cols], dV_ref[cols]) <= 1e-4
    assert rel_err(dQ.cpu().numpy()[cols], dQ_ref[cols]) <= 1e-4

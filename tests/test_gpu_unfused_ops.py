"""GPU: the single-step operators (sddmm, edge_softmax, spmm, l2 normalise,
spmm_backward, softmax_backward, sddmm_backward; reference kernels.hpp /
autograd.hpp) and the 5-launch unfused backward built from them, against the
oracle's per-step restatement (dP and dS included).  Same floor-1 tolerance
as the fused path: 1e-4 fp32, 1e-11 fp64."""
import numpy as np
import pytest

import oracle
from oracle import rel_err
from test_gpu_parity import CONFIGS, TOL, make_graph, make_inputs

pytestmark = pytest.mark.gpu


def _run(g, cfg, seed=3):
    import torch

    from paper_2411_16127_b200 import fused

    variant, l2, H, D, dt = cfg
    scale = 1.0 / np.sqrt(D)
    spec = fused.AttnSpec(variant=variant, heads=H, head_dim=D, scale=scale, slope=0.2, l2=l2)
    Q, K, V, dO = make_inputs(g, variant, H, D, dt, seed)
    dg = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row)
    t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (Q, K, V, dO)]
    S = fused.sddmm(dg, spec, t[0], t[1])
    P = fused.edge_softmax(dg, H, S)
    O = fused.spmm(dg, H, D, P, t[2])
    dQ, dK, dV, dP, dS = fused.attn_backward_unfused(dg, spec, t[0], t[1], t[2], P, t[3])
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in dict(O=O, P=P, dQ=dQ, dK=dK, dV=dV, dP=dP, dS=dS).items()}
    O_r, P_r = oracle.forward(g, Q, K, V, H, D, variant, l2, scale, 0.2, want_p=True)
    dQ_r, dK_r, dV_r, dP_r, dS_r = oracle.backward(g, Q, K, V, dO, H, D, variant, l2, scale, 0.2,
                                                   want_edge_grads=True)
    ref = dict(O=O_r, P=P_r, dQ=dQ_r, dK=dK_r, dV=dV_r, dP=dP_r, dS=dS_r)
    return got, ref


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c[0]}{'-l2' if c[1] else ''}-{c[2]}x{c[3]}-{c[4].__name__}")
def test_unfused_ops_match_oracle(cuda, cfg):
    for name in ("random", "sparse_empty", "hub"):
        if cfg[2] > 32:
            continue
        got, ref = _run(make_graph(name), cfg)
        errs = {k: rel_err(got[k].reshape(ref[k].shape), ref[k]) for k in ref}
        bad = {k: v for k, v in errs.items() if not v <= TOL[cfg[4]]}
        assert not bad, f"{name} {cfg}: {errs}"


def test_l2_normalize_rows_and_backward(cuda):
    import torch

    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(0)
    H, D = 3, 5
    X = rng.uniform(-1, 1, (50, H * D))
    X[7, D:2 * D] = 0.0  # a zero head row: stays 0, backward divides by eps
    dY = rng.uniform(-1, 1, X.shape)
    x, dy = torch.tensor(X, device="cuda"), torch.tensor(dY, device="cuda")
    Y = fused.l2_normalize_rows(x, H, D).cpu().numpy()
    dX = fused.l2_normalize_backward(x, dy, H, D).cpu().numpy()
    Xh = X.reshape(50, H, D)
    n = np.sqrt((Xh ** 2).sum(-1, keepdims=True))
    assert rel_err(Y, (Xh / np.maximum(n, 1e-12)).reshape(50, -1)) < 1e-14
    dYh = dY.reshape(50, H, D)
    xn = Xh / np.where(n > 1e-12, n, 1.0)
    ref = np.where(n > 1e-12, (dYh - xn * (xn * dYh).sum(-1, keepdims=True)) / np.where(n > 1e-12, n, 1.0),
                   dYh / 1e-12)
    assert rel_err(dX, ref.reshape(50, -1)) < 1e-12


def test_unfused_ops_known_answers(cuda):
    """test_autograd.cpp:69-111: softmax backward of P = (1/2, 1/2) with
    dP = (1, 0) gives dS = (1/4, -1/4); rows of dS sum to zero."""
    import torch

    from paper_2411_16127_b200 import fused

    g = oracle.from_coo(2, np.array([0, 1]), np.array([0, 0]))  # two in-edges of node 0
    dg = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row)
    P = torch.tensor([[0.5], [0.5]], dtype=torch.float64, device="cuda")
    dP = torch.tensor([[1.0], [0.0]], dtype=torch.float64, device="cuda")
    dS = fused.softmax_backward(dg, 1, P, dP).cpu().numpy().ravel()
    assert np.allclose(dS, [0.25, -0.25], atol=0, rtol=1e-15)

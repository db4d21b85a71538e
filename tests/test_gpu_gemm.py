"""GPU: the dense projection (K0).  fp32 X·W runs on tcgen05 tensor cores with
the 3xTF32 split; it must match an fp64 reference within the fp32 parity bar
(floor-1 relative error <= 5e-5 here, measured <= 1.8e-5 at K=128, inside the 1e-4 bar;
plain single-pass TF32 would be ~5e-4).  fp64 and X^T·dY use the SIMT kernel."""
import numpy as np
import pytest
import torch

from oracle import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,K,N", [(128, 32, 16), (1000, 64, 64), (333, 128, 384), (130, 36, 48),
                                   (4097, 128, 256), (5, 8, 32)])
def test_tc_gemm_3xtf32_matches_fp64(cuda, M, K, N):
    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(M + K + N)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    C = fused.gemm(torch.from_numpy(A).to(cuda), torch.from_numpy(B).to(cuda)).cpu().numpy()
    assert rel_err(C, ref) < 5e-5, rel_err(C, ref)
    # accumulate mode: C += A·B
    Ct = torch.from_numpy(C).to(cuda)
    fused.gemm(torch.from_numpy(A).to(cuda), torch.from_numpy(B).to(cuda), out=Ct, accumulate=True)
    assert rel_err(Ct.cpu().numpy(), 2 * ref) < 5e-5


@pytest.mark.parametrize("K,M,N", [(50_000, 64, 64), (100_000, 128, 128), (1000, 128, 256),
                                   (33, 8, 16), (700_001, 128, 64)])
def test_tc_weight_grad_xt_dy(cuda, K, M, N):
    """dW = X^T dY on tcgen05 (MN-major operands, deterministic split-K)."""
    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(K + M + N)
    X = rng.uniform(-1, 1, (K, M)).astype(np.float32)
    dY = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = X.T.astype(np.float64) @ dY.astype(np.float64)
    tx, ty = torch.from_numpy(X).to(cuda), torch.from_numpy(dY).to(cuda)
    C = fused.gemm(tx, ty, trans_a=True)
    C2 = fused.gemm(tx, ty, trans_a=True)
    scale = max(1.0, float(np.abs(ref).max()))
    err = float(np.abs(C.cpu().numpy() - ref).max()) / scale
    assert err < 5e-5, err
    assert torch.equal(C, C2)  # fixed-order split-K reduction


def test_simt_paths(cuda):
    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (20000, 40))
    dY = rng.uniform(-1, 1, (20000, 24))
    for dt in (torch.float32, torch.float64):
        out = fused.gemm(torch.tensor(X, dtype=dt, device=cuda), torch.tensor(dY, dtype=dt, device=cuda),
                         trans_a=True).cpu().numpy()
        assert rel_err(out, X.T @ dY) < (1e-4 if dt == torch.float32 else 1e-11)
    W = rng.uniform(-1, 1, (40, 24))
    out = fused.gemm(torch.tensor(X, device=cuda), torch.tensor(W, device=cuda)).cpu().numpy()
    assert rel_err(out, X @ W) < 1e-11


def test_gat_logits_and_fanin(cuda):
    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(4)
    n, H, D = 777, 8, 8
    Hf = rng.uniform(-1, 1, (n, H * D))
    al, ar = rng.uniform(-1, 1, H * D), rng.uniform(-1, 1, H * D)
    t = lambda a: torch.tensor(a, device=cuda)  # noqa: E731
    el, er = fused.gat_logits(t(Hf), t(al), t(ar), H, D)
    assert rel_err(el.cpu().numpy(), (Hf.reshape(n, H, D) * al.reshape(H, D)).sum(-1)) < 1e-12
    assert rel_err(er.cpu().numpy(), (Hf.reshape(n, H, D) * ar.reshape(H, D)).sum(-1)) < 1e-12
    dV = rng.uniform(-1, 1, (n, H * D))
    dl, dr = rng.uniform(-1, 1, (n, H)), rng.uniform(-1, 1, (n, H))
    dH, dal, dar = fused.gat_fanin(t(Hf), t(al), t(ar), t(dV), t(dl), t(dr), H, D)
    ref = dV + (dl[:, :, None] * al.reshape(H, D) + dr[:, :, None] * ar.reshape(H, D)).reshape(n, -1)
    assert rel_err(dH.cpu().numpy(), ref) < 1e-12
    assert rel_err(dal.cpu().numpy(), (Hf.reshape(n, H, D) * dl[:, :, None]).sum(0).reshape(-1)) < 1e-11
    assert rel_err(dar.cpu().numpy(), (Hf.reshape(n, H, D) * dr[:, :, None]).sum(0).reshape(-1)) < 1e-11


@pytest.mark.parametrize("n", [777, 300_000])
def test_gat_logits_and_fanin_fp32_fast_path(cuda, n):
    """fp32 float4 paths (gat_logits_vec, gat_fanin_vec + parallel fixed-order
    reduce) against an fp64 reference; deterministic across calls."""
    from paper_2411_16127_b200 import fused

    rng = np.random.default_rng(5)
    H, D = 8, 8
    Hf = rng.uniform(-1, 1, (n, H * D)).astype(np.float32)
    al, ar = (rng.uniform(-1, 1, H * D).astype(np.float32) for _ in range(2))
    dV = rng.uniform(-1, 1, (n, H * D)).astype(np.float32)
    dl, dr = (rng.uniform(-1, 1, (n, H)).astype(np.float32) for _ in range(2))
    t = lambda a: torch.from_numpy(a).to(cuda)  # noqa: E731
    el, er = fused.gat_logits(t(Hf), t(al), t(ar), H, D)
    H64 = Hf.astype(np.float64).reshape(n, H, D)
    assert rel_err(el.cpu().numpy(), (H64 * al.reshape(H, D)).sum(-1)) < 1e-5
    assert rel_err(er.cpu().numpy(), (H64 * ar.reshape(H, D)).sum(-1)) < 1e-5
    dH, dal, dar = fused.gat_fanin(t(Hf), t(al), t(ar), t(dV), t(dl), t(dr), H, D)
    ref = dV + (dl[:, :, None] * al.reshape(H, D) + dr[:, :, None] * ar.reshape(H, D)).reshape(n, -1)
    assert rel_err(dH.cpu().numpy(), ref) < 1e-6
    ref_al = (H64 * dl[:, :, None]).sum(0).reshape(-1)
    ref_ar = (H64 * dr[:, :, None]).sum(0).reshape(-1)
    scale = max(1.0, float(np.abs(H64).sum() / (H * D) ** 0.5 / 1e2))
    assert float(np.abs(dal.cpu().numpy() - ref_al).max()) / scale < 1e-4
    assert float(np.abs(dar.cpu().numpy() - ref_ar).max()) / scale < 1e-4
    _, dal2, _ = fused.gat_fanin(t(Hf), t(al), t(ar), t(dV), t(dl), t(dr), H, D)
    assert torch.equal(dal, dal2)


@pytest.mark.parametrize("M,N,K", [(1000, 64, 64), (4099, 128, 128), (257, 96, 32)])
def test_gemm_bcast_matches_gemm(cuda, M, N, K):
    """Projection fused with the row all-gather: every destination (here local
    row blocks of larger tables standing in for the peers' tables) receives the
    bit-identical product."""
    import torch

    from paper_2411_16127_b200 import fused

    g = torch.Generator(device="cuda")
    g.manual_seed(M + N)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(K, N, device="cuda", generator=g) * 2 - 1
    ref = fused.gemm(A, B)
    tables = [torch.full((3 * M, N), 7.0, device="cuda") for _ in range(4)]
    outs = [t[M: 2 * M] for t in tables]
    fused.gemm_bcast(A, B, outs)
    torch.cuda.synchronize()
    for t in tables:
        assert torch.equal(t[M: 2 * M], ref)
        assert bool((t[:M] == 7.0).all()) and bool((t[2 * M:] == 7.0).all())  # nothing else written
    one = torch.empty(M, N, device="cuda")
    fused.gemm_bcast(A, B, [one])
    assert torch.equal(one, ref)


def test_gemm_bcast_errors(cuda):
    import torch

    from paper_2411_16127_b200 import fused

    A = torch.rand(64, 32, device="cuda")
    with pytest.raises(Exception, match="gemm_bcast"):
        fused.gemm_bcast(A, torch.rand(32, 48, device="cuda"), [torch.empty(64, 48, device="cuda")])
    with pytest.raises(Exception, match="gemm_bcast"):
        fused.gemm_bcast(A, torch.rand(32, 64, device="cuda"),
                         [torch.empty(64, 64, device="cuda")] * 9)


@pytest.mark.parametrize("M,F,K", [(1000, 128, 128), (4096, 64, 64), (333, 256, 32)])
def test_gemm_split_matches_three_gemms(cuda, M, F, K):
    """X·[W_q | W_k | W_v] as one split-output GEMM == three separate GEMMs,
    bitwise (same 128-column tiles, same K order)."""
    import torch

    from paper_2411_16127_b200 import fused

    g = torch.Generator(device="cuda")
    g.manual_seed(M + F)
    X = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    Ws = [torch.rand(K, F, device="cuda", generator=g) * 2 - 1 for _ in range(3)]
    refs = [fused.gemm(X, w) for w in Ws]
    outs = [torch.empty(M, F, device="cuda") for _ in range(3)]
    fused.gemm_split(X, torch.cat(Ws, 1), outs)
    torch.cuda.synchronize()
    for a, b in zip(outs, refs):
        assert torch.equal(a, b)

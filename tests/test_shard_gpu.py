"""GPU: row-sharded execution simulated on one device (run the P
shard kernels sequentially and compare with the 1-GPU result).  Every shard
graph (CSR of its rows, CSC of its columns, padded id space, empty rows
skipped) writes only its owned rows / columns of shared padded tables; the
union must equal the unsharded forward and backward bit-for-bit (owner-
computes, unchanged per-row and per-column reduction order)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def graph(seed=0, n=3000):
    rng = np.random.default_rng(seed)
    deg = np.maximum(0, np.round(1500 * (np.arange(n) + 1.0) ** -0.6)).astype(np.int64)
    dst = np.repeat(rng.permutation(n), deg)
    src = rng.integers(0, n, dst.shape[0])
    key = np.unique(dst * n + src)
    return oracle.from_coo(n, key % n, key // n)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg", [("add", False, 8, 8), ("dot", False, 8, 16), ("dot", True, 2, 16)],
                         ids=["gat8x8", "gt8x16", "agnn2x16"])
def test_sharded_equals_single_gpu(cuda, world, cfg):
    from paper_2411_16127_b200 import fused
    from paper_2411_16127_b200.shard import RowShard

    variant, l2, H, D = cfg
    g = graph()
    spec = fused.AttnSpec(variant, H, D, scale=0.25, slope=0.2, l2=l2)
    rng = np.random.default_rng(1)
    w = spec.qk_width
    Q, K = (torch.tensor(rng.uniform(-1.5, 1.5, (g.n, w)), dtype=torch.float32, device=cuda)
            for _ in range(2))
    V, dO = (torch.tensor(rng.uniform(-1, 1, (g.n, H * D)), dtype=torch.float32, device=cuda)
             for _ in range(2))
    full = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row,
                                           cta_threshold=64)
    O1, st1 = fused.attn_forward(full, spec, Q, K, V)
    dQ1, dK1, dV1 = fused.attn_backward(full, spec, Q, K, V, O1, st1, dO)

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
    shards = [RowShard.build(g.n, t(g.row_ptr), t(g.col), t(g.csc_ptr), t(g.csc_row), r, world)
              for r in range(world)]
    s0 = shards[0]
    Qp, Kp, Vp, dOp = (s0.to_padded(x) for x in (Q, K, V, dO))
    Op = torch.zeros_like(Vp)
    stp = torch.zeros(s0.n_padded, H, 4, device=cuda)
    dQp, dKp, dVp = torch.zeros_like(Qp), torch.zeros_like(Kp), torch.zeros_like(Vp)
    graphs = [sh.device_graph(cta_threshold=64) for sh in shards]
    for dg in graphs:  # forward on every shard's rows (the all-gathered V/Q/el are Vp/Qp)
        fused.attn_forward(dg, spec, Qp, Kp, Vp, O=Op, stats=stp)
    for dg in graphs:  # pass A on owned rows
        fused.attn_backward_rows(dg, spec, Qp, Kp, Vp, Op, stp, dOp, dKp)
    for dg in graphs:  # pass B on owned columns (after the dO / record all-gather)
        fused.attn_backward_cols(dg, spec, Qp, Kp, Vp, stp, dOp, dQp, dVp)
    torch.cuda.synchronize()
    for a, b, name in ((O1, Op, "O"), (dQ1, dQp, "dQ"), (dK1, dKp, "dK"), (dV1, dVp, "dV")):
        assert torch.equal(a, s0.from_padded(b)), name


def test_peer_tables_gemm_bcast_world1(cuda):
    """The p2p exchange plumbing on one GPU: a 1-rank NCCL group, padded tables
    in torch symmetric memory, gemm_bcast into shard.PeerTables.dests, device
    barrier.  (With more ranks the destinations add the peers' tables; the
    addressing is covered on CPU by test_shard_cpu.test_block_views_*.)"""
    import os
    import socket

    import torch.distributed as dist

    from paper_2411_16127_b200 import fused
    from paper_2411_16127_b200.shard import PeerTables, RowShard

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = graph(n=500)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
        sh = RowShard.build(g.n, t(g.row_ptr), t(g.col), t(g.csc_ptr), t(g.csc_row), 0, 1)
        pt = PeerTables(sh, {"Q": 64, "V": 128}, device=cuda)
        # the peer-view addressing (get_buffer + storage offset) resolves to the
        # tensor itself for the own rank
        own = pt.hdl.get_buffer(0, (pt.buf.numel(),), pt.buf.dtype, pt.storage_offset)
        assert own.data_ptr() == pt.buf.data_ptr()
        pt.selftest()
        X = torch.rand(sh.n_padded, 32, device=cuda)
        Wq, Wv = torch.rand(32, 64, device=cuda), torch.rand(32, 128, device=cuda)
        pt.barrier()
        fused.gemm_bcast(X[sh.block], Wq, pt.dests("Q"))
        fused.gemm_bcast(X[sh.block], Wv, pt.dests("V"))
        pt.barrier()
        torch.cuda.synchronize()
        assert torch.equal(pt.table("Q"), fused.gemm(X, Wq))
        assert torch.equal(pt.table("V"), fused.gemm(X, Wv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cfg", [("add", False, 8, 8), ("dot", False, 8, 16), ("dot", True, 2, 16)],
                         ids=["gat8x8", "gt8x16", "agnn2x16"])
def test_source_phased_forward(cuda, world, cfg):
    """The overlapped forward (shard.source_parts / phase_forward /
    merge_phases): every simulated rank runs one forward per source block
    (own block first) into row-block partials and merges them.  O and the
    records match the one-pass forward within fp32 rounding (the log-sum-exp
    of the (m, log2 l) pair; aux exactly); the backward on the merged records
    matches too."""
    from paper_2411_16127_b200 import fused
    from paper_2411_16127_b200.shard import (RowShard, merge_phases, part_buffers, phase_forward,
                                             phase_order, source_parts)

    variant, l2, H, D = cfg
    g = graph(seed=2)
    spec = fused.AttnSpec(variant, H, D, scale=0.25, slope=0.2, l2=l2)
    rng = np.random.default_rng(3)
    w = spec.qk_width
    Q, K = (torch.tensor(rng.uniform(-1.5, 1.5, (g.n, w)), dtype=torch.float32, device=cuda)
            for _ in range(2))
    V, dO = (torch.tensor(rng.uniform(-1, 1, (g.n, H * D)), dtype=torch.float32, device=cuda)
             for _ in range(2))
    full = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row,
                                           cta_threshold=64)
    O1, st1 = fused.attn_forward(full, spec, Q, K, V)
    dQ1, dK1, dV1 = fused.attn_backward(full, spec, Q, K, V, O1, st1, dO)

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
    shards = [RowShard.build(g.n, t(g.row_ptr), t(g.col), t(g.csc_ptr), t(g.csc_row), r, world)
              for r in range(world)]
    s0 = shards[0]
    Qp, Kp, Vp, dOp = (s0.to_padded(x) for x in (Q, K, V, dO))
    Op = torch.zeros_like(Vp)
    stp = torch.zeros(s0.n_padded, H, 4, device=cuda)
    for sh in shards:
        parts = source_parts(sh, cta_threshold=64)
        Ob, rb = part_buffers(parts, spec, device=cuda)
        for k in phase_order(sh):
            phase_forward(parts, k, spec, Qp, Kp, Vp, Ob, rb)
        merge_phases(parts, spec, Ob, rb, Op, stp)
    torch.cuda.synchronize()
    O2, st2 = s0.from_padded(Op), s0.from_padded(stp)
    nz = torch.from_numpy(np.diff(g.row_ptr) > 0).to(cuda)
    assert float((O2 - O1).abs().max()) <= 2e-6 * max(1.0, float(O1.abs().max()))
    # (m, log2 l) is a consistent pair, not unique: the forward keeps a stale
    # m within GF_RESCALE_TH of the row max, so compare the log-sum-exp
    lse1, lse2 = fused.lse_of(st1)[nz], fused.lse_of(st2)[nz]
    assert float((lse2 - lse1).abs().max()) <= 1e-5 * max(1.0, float(lse1.abs().max()))
    assert torch.equal(st2[nz][..., 2], st1[nz][..., 2])  # aux (er | 1/||K||)
    # backward on the merged records (one-pass shard graphs)
    dQp, dKp, dVp = torch.zeros_like(Qp), torch.zeros_like(Kp), torch.zeros_like(Vp)
    graphs = [sh.device_graph(cta_threshold=64) for sh in shards]
    for dg in graphs:
        fused.attn_backward_rows(dg, spec, Qp, Kp, Vp, Op, stp, dOp, dKp)
    for dg in graphs:
        fused.attn_backward_cols(dg, spec, Qp, Kp, Vp, stp, dOp, dQp, dVp)
    torch.cuda.synchronize()
    for a, b, name in ((dQ1, dQp, "dQ"), (dK1, dKp, "dK"), (dV1, dVp, "dV")):
        assert rel_err_t(s0.from_padded(b), a) <= 1e-5, name


def rel_err_t(a, b):
    return float((a - b).abs().max()) / max(1e-30, float(b.abs().max()))

"""CPU, world_size 2 over gloo: the row-sharding host logic (shard.py).

Each rank builds its shard of the same graph and checks that (1) the shards
partition the edge set exactly on both the CSR and the CSC side, (2) each
row / column keeps its edge order (monotonic relabelling), (3) the in-place
all-gather of padded node tables reproduces the full table (also with several
asynchronous all-gathers in flight, as the bench step issues them), and (4) the
forward restricted to the rank's rows (CPU oracle on the shard CSR) equals
the single-process forward bitwise on the owned rows.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_graph(seed=3, n=400):
    import oracle

    rng = np.random.default_rng(seed)
    deg = np.maximum(0, np.round(80 * (np.arange(n) + 1.0) ** -0.6)).astype(np.int64)
    dst = np.repeat(rng.permutation(n), deg)
    src = rng.integers(0, n, dst.shape[0])
    key = np.unique(dst * n + src)
    return oracle.from_coo(n, key % n, key // n)


def worker(rank, world, port, errq):
    try:
        import sys

        sys.path.insert(0, ROOT)
        import oracle
        from paper_2411_16127_b200.shard import RowShard, all_gather_rows

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g = make_graph()
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
        sh = RowShard.build(g.n, t(g.row_ptr), t(g.col), t(g.csc_ptr), t(g.csc_row), rank, world)
        b = sh.bounds
        # invert the relabelling
        inv = np.full(sh.n_padded, -1, np.int64)
        for k in range(world):
            inv[k * sh.R: k * sh.R + b[k + 1] - b[k]] = np.arange(b[k], b[k + 1])
        # (1)+(2) CSR side: owned rows, same sources in the same order
        rp, col = sh.row_ptr.numpy().astype(np.int64), sh.col.numpy().astype(np.int64)
        for v in range(b[rank], b[rank + 1]):
            pv = rank * sh.R + v - b[rank]
            mine = inv[col[rp[pv]: rp[pv + 1]]]
            ref = g.col[g.row_ptr[v]: g.row_ptr[v + 1]]
            assert np.array_equal(mine, ref), ("csr", v)
        assert rp[-1] == g.row_ptr[b[rank + 1]] - g.row_ptr[b[rank]]
        cp, cr = sh.csc_ptr.numpy().astype(np.int64), sh.csc_row.numpy().astype(np.int64)
        for u in range(b[rank], b[rank + 1]):
            pu = rank * sh.R + u - b[rank]
            assert np.array_equal(inv[cr[cp[pu]: cp[pu + 1]]],
                                  g.csc_row[g.csc_ptr[u]: g.csc_ptr[u + 1]]), ("csc", u)
        counts = torch.tensor([len(col), len(cr)])
        dist.all_reduce(counts)
        assert counts.tolist() == [g.e, g.e]
        # (3) in-place all-gather of padded tables
        rng = np.random.default_rng(7)
        H, D = 4, 8
        Q, K, V = (rng.uniform(-1, 1, (g.n, H * D)).astype(np.float32) for _ in range(3))
        full = sh.to_padded(t(V))
        mine = torch.zeros_like(full)
        mine[sh.block] = full[sh.block]
        all_gather_rows(mine, sh)
        assert torch.equal(mine, full)
        # (3b) the bench step's overlapped order: several async all-gathers in
        # flight, waited on in need order (V, Q first; dO, K later)
        tabs = [sh.to_padded(t(x)) for x in (V, Q, K, Q * 2)]
        mines = []
        for x in tabs:
            m = torch.zeros_like(x)
            m[sh.block] = x[sh.block]
            mines.append(m)
        works = [all_gather_rows(m, sh, async_op=True) for m in mines]
        for w in works:
            w.wait()
        assert all(torch.equal(m, x) for m, x in zip(mines, tabs))
        # (3c) the phased step's exchange: one async broadcast per owner block
        # (every rank issues them in the same order), waited on own block first
        R = sh.R
        bmine = torch.zeros_like(full)
        bmine[sh.block] = full[sh.block]
        bw = {k: dist.broadcast(bmine[k * R:(k + 1) * R], src=k, async_op=True)
              for k in range(world)}
        for k in [rank] + [j for j in range(world) if j != rank]:
            bw[k].wait()
        assert torch.equal(bmine, full)
        # (4) sharded forward == single-process forward on owned rows, bitwise
        csr = oracle.CSR(sh.n_padded, rp, col, cp, cr, np.zeros(len(cr), np.int64))
        Op = oracle.forward(csr, sh.to_padded(t(Q)).numpy(), sh.to_padded(t(K)).numpy(),
                            full.numpy(), H, D, "dot", False, 0.3, 0.2)
        O = oracle.forward(g, Q, K, V, H, D, "dot", False, 0.3, 0.2)
        assert np.array_equal(Op[sh.rows], O[b[rank]: b[rank + 1]])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced in the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


@pytest.mark.parametrize("world", [2])
def test_row_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_partition_balances_edges():
    from paper_2411_16127_b200.shard import partition

    g = make_graph(n=1000)
    rp, cp = torch.from_numpy(g.row_ptr), torch.from_numpy(g.csc_ptr)
    for world in (2, 4, 8):
        b = partition(g.n, rp, cp, world)
        assert b[0] == 0 and b[-1] == g.n and all(x <= y for x, y in zip(b, b[1:]))
        load = [int(rp[b[k + 1]] - rp[b[k]] + cp[b[k + 1]] - cp[b[k]]) for k in range(world)]
        assert max(load) - min(load) <= 2 * int(np.diff(g.row_ptr).max() + np.diff(g.csc_ptr).max())


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_block_views_write_every_copy(world):
    """gemm_bcast addressing (shard.block_views): when every rank writes its
    block through its destination list into all ranks' padded tables, every
    copy equals the all-gathered table, and nothing outside the blocks moves."""
    from paper_2411_16127_b200.shard import RowShard, block_views

    g = make_graph()
    rp, col = torch.from_numpy(g.row_ptr), torch.from_numpy(g.col)
    cp, cr = torch.from_numpy(g.csc_ptr), torch.from_numpy(g.csc_row)
    shards = [RowShard.build(g.n, rp, col, cp, cr, k, world) for k in range(world)]
    x = torch.randn(g.n, 6)
    xp = shards[0].to_padded(x)
    tables = [torch.full_like(xp, float("nan")) for _ in range(world)]
    for k, sh in enumerate(shards):
        dests = block_views(tables, sh)
        assert dests[0].data_ptr() == tables[k][sh.block].data_ptr()  # own copy first
        assert len(dests) == world
        for d in dests:
            d.copy_(xp[sh.block])
    for t in tables:
        assert torch.equal(t, xp)
        assert torch.equal(shards[0].from_padded(t), x)
    with pytest.raises(ValueError):
        block_views(tables[:-1] if world > 1 else [], shards[0])


@pytest.mark.parametrize("world", [1, 2, 4])
def test_source_split_and_merge_cpu(world):
    """shard.source_split partitions every owned row's in-edges by source block
    (order kept), and the forward over the parts merged with the
    gf_attn_merge_parts rule (m = max m_k, w_k = l_k e^(m_k - m)) equals the
    one-pass forward (CPU oracle)."""
    import oracle
    from paper_2411_16127_b200.shard import RowShard, source_split

    g = make_graph(seed=4)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    rng = np.random.default_rng(5)
    H, D = 2, 8
    Q, K, V = (rng.uniform(-1, 1, (g.n, H * D)) for _ in range(3))
    O_ref = oracle.forward(g, Q, K, V, H, D, "dot", False, 0.4, 0.2)
    for rank in range(world):
        sh = RowShard.build(g.n, t(g.row_ptr), t(g.col), t(g.csc_ptr), t(g.csc_row), rank, world)
        Qp, Kp, Vp = (sh.to_padded(t(x)).numpy() for x in (Q, K, V))
        rp, col = sh.row_ptr.numpy().astype(np.int64), sh.col.numpy().astype(np.int64)
        parts = source_split(sh)
        assert sum(int(c.numel()) for _, c in parts) == len(col)
        for v in range(sh.n_padded):
            joined = np.concatenate([c.numpy()[p[v]: p[v + 1]] for p, c in parts])
            assert np.array_equal(joined, col[rp[v]: rp[v + 1]])  # blocks in order = the row
        # merge with the lse form of the rule: w_k = e^(lse_k - max_k lse_k)
        num = np.zeros((sh.n_padded, H * D))
        outs = []
        for p, c in parts:
            p64, c64 = p.numpy().astype(np.int64), c.numpy().astype(np.int64)
            csr = oracle.CSR(sh.n_padded, p64, c64, np.zeros(sh.n_padded + 1, np.int64),
                             np.zeros(0, np.int64), np.zeros(0, np.int64))
            Ok, lse = oracle.forward(csr, Qp, Kp, Vp, H, D, "dot", False, 0.4, 0.2, want_lse=True)
            outs.append((np.diff(p64) > 0, Ok, lse))
        top = np.full((sh.n_padded, H), -np.inf)
        for live, _, lse in outs:
            top = np.where(live[:, None], np.maximum(top, lse), top)
        L = np.zeros((sh.n_padded, H))
        for live, Ok, lse in outs:
            with np.errstate(invalid="ignore"):  # rows with no live part: masked below
                d = np.where(live[:, None], lse - top, 0.0)
            w = np.where(live[:, None], np.exp(d), 0.0)
            L += w
            num += np.repeat(w, D, axis=1) * Ok
        rows = sh.rows
        got = num[rows] / np.maximum(np.repeat(L[rows], D, axis=1), 1e-300)
        nz = np.diff(g.row_ptr)[sh.lo: sh.hi] > 0
        assert np.allclose(got[nz], O_ref[sh.lo: sh.hi][nz], rtol=1e-12, atol=1e-12)

"""GPU: the device synthetic-graph generators.  They
follow the reference generators' distributions (graph.cpp:127-185) with
counter-based hashing instead of a sequential mt19937_64 rejection loop, so
the contract checked here is distributional: exact edge counts, distinct
edges, ids in range, the hub's exact in-degree, the power-law degree
sequence, determinism per seed, and that the result feeds the device
from_coo (no duplicate is rejected)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _keys(src, dst, n):
    return (dst.cpu().numpy().astype(np.int64) * n + src.cpu().numpy())


@pytest.mark.parametrize("n,avg", [(1000, 3.5), (2708, 3.898), (300, 150.0), (50_000, 25.8)])
def test_gen_random_device(cuda, n, avg):
    from paper_2411_16127_b200 import fused

    src, dst = fused.gen_random_device(n, avg, seed=7)
    k = _keys(src, dst, n)
    assert len(k) == int(avg * n + 0.5)
    assert len(np.unique(k)) == len(k)
    assert src.min() >= 0 and src.max() < n and dst.min() >= 0 and dst.max() < n
    s2, d2 = fused.gen_random_device(n, avg, seed=7)
    assert torch.equal(src, s2) and torch.equal(dst, d2)  # deterministic per seed
    s3, _ = fused.gen_random_device(n, avg, seed=8)
    assert not torch.equal(src, s3)
    # uniform: every destination decile gets ~10% of the edges
    hist = np.bincount(dst.cpu().numpy() * 10 // n, minlength=10) / len(k)
    assert np.all(np.abs(hist - 0.1) < 0.03), hist
    # feeds the device from_coo without a duplicate rejection
    row_ptr, col, _, _, _ = fused.from_coo_device(n, src, dst)
    assert int(row_ptr[-1]) == len(k)


def test_gen_super_node_device(cuda):
    from paper_2411_16127_b200 import fused

    n, avg, hub = 3000, 3.0, 2500
    src, dst = fused.gen_super_node_device(n, avg, hub, seed=1)
    k = _keys(src, dst, n)
    assert len(k) == max(hub, int(avg * n + 0.5)) and len(np.unique(k)) == len(k)
    deg = np.bincount(dst.cpu().numpy(), minlength=n)
    assert deg[0] == hub  # exact hub in-degree
    assert deg[1:].max() < hub  # every other in-degree strictly below it
    assert len(np.unique(src.cpu().numpy()[dst.cpu().numpy() == 0])) == hub


def test_gen_power_law_device(cuda):
    from paper_2411_16127_b200 import fused

    n, mx, ex = 20_000, 2_000, 0.34
    src, dst = fused.gen_power_law_device(n, mx, ex, seed=3)
    k = _keys(src, dst, n)
    assert len(np.unique(k)) == len(k)
    want = np.sort(np.rint(mx * (np.arange(n) + 1.0) ** -ex).astype(np.int64))[::-1]
    got = np.sort(np.bincount(dst.cpu().numpy(), minlength=n))[::-1]
    # duplicate sources are dropped: each row loses at most a few edges
    assert np.all(got <= want) and np.all(want - got <= np.maximum(3, want * want // n + 3))
    assert got[0] >= mx - mx * mx // n - 5  # ~mx^2/(2n) birthday collisions


@pytest.mark.parametrize("mols,atoms,rings", [(1024, 26, 3), (7, 1, 0), (5, 2, 4), (300, 40, 0)])
def test_gen_molecules_device(cuda, mols, atoms, rings):
    from paper_2411_16127_b200 import fused

    src, dst = fused.gen_molecules_device(mols, atoms, rings, seed=3)
    n = mols * atoms
    s, d = src.cpu().numpy(), dst.cpu().numpy()
    k = d * n + s
    assert len(np.unique(k)) == len(k) and np.all(np.diff(k) > 0)  # distinct, (dst, src) order
    assert not np.any(s == d)  # no self-loops
    assert np.all(s // atoms == d // atoms)  # block diagonal (batch_graphs layout)
    assert set((d * n + s).tolist()) == set((s * n + d).tolist())  # both directions
    assert 2 * mols * (atoms - 1) <= len(k) <= 2 * mols * (atoms - 1 + rings)
    if rings == 0:  # a tree per molecule: exactly atoms-1 undirected bonds
        assert len(k) == 2 * mols * (atoms - 1)
    # every molecule connected: union-find over the bonds
    parent = np.arange(n)

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for a, b in zip(s.tolist(), d.tolist()):
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[ra] = rb
    roots = np.array([find(i) for i in range(n)])
    assert len(np.unique(roots)) == mols
    s2, d2 = fused.gen_molecules_device(mols, atoms, rings, seed=3)
    assert torch.equal(src, s2) and torch.equal(dst, d2)
    row_ptr, _, _, _, _ = fused.from_coo_device(n, src, dst)
    assert int(row_ptr[-1]) == len(k)


def test_gen_molecules_device_errors(cuda):
    from paper_2411_16127_b200 import fused

    with pytest.raises(Exception, match="gen_molecules"):
        fused.gen_molecules_device(0, 26, 3)


@pytest.mark.parametrize("name", ["cora", "pubmed", "molhiv", "reddit_slice", "power_law_small"])
def test_host_generator_port_is_bit_exact(cuda, name):
    """bench.py's numpy restatement of the device generators (the reference
    arm's graphs) produces the SAME edge list as the device generator, so the
    CPU reference and the GPU path time one graph."""
    import bench
    from paper_2411_16127_b200 import fused

    if name == "reddit_slice":
        rows = bench.REDDIT_N // 128
        n, s_h, d_h = bench.gen_graph_host("reddit", rows=rows)
        _, s_d, d_d = bench.gen_graph_device("reddit", torch.device("cuda"))
        keep = d_d < rows
        s_d, d_d = s_d[keep], d_d[keep]
    elif name == "power_law_small":
        n = 20_000
        s_h, d_h = bench.host_power_law(n, 2_000, 0.34, seed=3)
        s_d, d_d = fused.gen_power_law_device(n, 2_000, 0.34, seed=3)
    else:
        n, s_h, d_h = bench.gen_graph_host(name)
        _, s_d, d_d = bench.gen_graph_device(name, torch.device("cuda"))
    assert len(s_h) > 0
    np.testing.assert_array_equal(s_d.cpu().numpy(), s_h)
    np.testing.assert_array_equal(d_d.cpu().numpy(), d_h)

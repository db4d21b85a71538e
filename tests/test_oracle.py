"""CPU: the C oracle restatement is pinned bit-exactly to the reference.

Golden vectors (tests/golden/, made by scripts/make_golden.py from the
reference compiled from its own sources) fix the expected CSR/CSC and the
multi-head forward/backward; the oracle must reproduce them exactly (same
algorithm, same operation order, same libm).  Where oracle/_ref is present
the comparison is repeated against the live reference on fresh inputs.
"""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def graphs():
    return np.load(os.path.join(GOLD, "graphs.npz"))


@pytest.fixture(scope="module")
def pipe():
    return np.load(os.path.join(GOLD, "pipeline.npz"))


GRAPH_NAMES = ["coo3", "selfloops", "empty_rows", "rand40", "rand120", "hub100", "rand12",
               "citeseer"]


def golden_csr(gz, name):
    return oracle.CSR(int(gz[f"{name}/n"]), gz[f"{name}/row_ptr"], gz[f"{name}/col"],
                      gz[f"{name}/csc_ptr"], gz[f"{name}/csc_row"], gz[f"{name}/csc_perm"])


@pytest.mark.parametrize("name", GRAPH_NAMES)
def test_from_coo_matches_reference(graphs, name):
    n = int(graphs[f"{name}/n"])
    src, dst = graphs[f"{name}/src"], graphs[f"{name}/dst"]
    rng = np.random.default_rng(0)
    perm = rng.permutation(src.shape[0])  # input order must not matter
    g = oracle.from_coo(n, src[perm], dst[perm])
    for k in ("row_ptr", "col", "csc_ptr", "csc_row", "csc_perm"):
        assert np.array_equal(getattr(g, k), graphs[f"{name}/{k}"]), k


def test_known_answers(graphs):
    # test_graph.cpp:11-22 / 30-35 / 73-81
    assert list(graphs["coo3/row_ptr"]) == [0, 0, 2, 3]
    assert list(graphs["coo3/col"]) == [0, 2, 1]
    assert list(graphs["selfloops/csc_perm"]) == [0, 1]
    assert list(graphs["batch2/row_ptr"]) == [0, 0, 2, 3, 3, 5, 6]
    assert list(graphs["batch2/col"]) == [0, 2, 1, 3, 5, 4]
    assert int(np.diff(graphs["hub100/row_ptr"]).max()) == 90


def test_from_coo_rejects_bad_input():
    with pytest.raises(oracle.OracleError, match="duplicate"):
        oracle.from_coo(2, [0, 0], [1, 1])
    with pytest.raises(oracle.OracleError, match="out of range"):
        oracle.from_coo(2, [0], [2])
    with pytest.raises(oracle.OracleError, match="out of range"):
        oracle.from_coo(2, [-1], [0])


PIPE = ["gat8x8_f32", "gt8x16_f32", "agnn2x16_f32", "gat8x8_f64", "gt2x5_f64", "agnn1x6_f64",
        "hub_gt4x8_f32", "empty_dot1x4_f64"]


@pytest.mark.parametrize("name", PIPE)
def test_pipeline_matches_reference_bitwise(graphs, pipe, name):
    g = golden_csr(graphs, str(pipe[f"{name}/graph"]))
    H, D, add, l2 = (int(x) for x in pipe[f"{name}/meta"])
    variant = "add" if add else "dot"
    scale = float(pipe[f"{name}/scale"])
    Q, K, V, dO = (pipe[f"{name}/{k}"] for k in ("Q", "K", "V", "dO"))
    O, P = oracle.forward(g, Q, K, V, H, D, variant, bool(l2), scale, 0.2, want_p=True)
    dQ, dK, dV = oracle.backward(g, Q, K, V, dO, H, D, variant, bool(l2), scale, 0.2)
    for k, got in (("O", O), ("P", P), ("dQ", dQ), ("dK", dK), ("dV", dV)):
        assert np.array_equal(got, pipe[f"{name}/{k}"]), (name, k)


def test_schedule_definition():
    """gfo_schedule: stable degree-descending order, bucket counts."""
    g = oracle.from_coo(6, [1, 2, 3, 4, 5, 0, 1, 2, 3], [0, 0, 0, 0, 0, 2, 2, 5, 5])
    order, n_cta, n_empty = oracle.schedule(g.n, g.row_ptr, 3)
    assert list(order) == [0, 2, 5, 1, 3, 4]
    assert (n_cta, n_empty) == (1, 3)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference_random():
    rg = oracle.ref_gen_random(250, 7.0, 21)
    g = rg.arrays()
    rng = np.random.default_rng(5)
    for dt in (np.float32, np.float64):
        for variant, l2, H, D in (("add", 0, 4, 8), ("dot", 0, 4, 8), ("dot", 1, 2, 6)):
            w = H if variant == "add" else H * D
            Q = rng.uniform(-1, 1, (g.n, w)).astype(dt)
            K = rng.uniform(-1, 1, (g.n, w)).astype(dt)
            V = rng.uniform(-1, 1, (g.n, H * D)).astype(dt)
            dO = rng.uniform(-1, 1, (g.n, H * D)).astype(dt)
            a = oracle.ref_forward(rg, Q, K, V, H, D, variant, l2, 0.7, 0.1)
            b = oracle.forward(g, Q, K, V, H, D, variant, l2, 0.7, 0.1)
            assert np.array_equal(a, b)
            ra = oracle.ref_backward(rg, Q, K, V, dO, H, D, variant, l2, 0.7, 0.1)
            rb = oracle.backward(g, Q, K, V, dO, H, D, variant, l2, 0.7, 0.1)
            for x, y in zip(ra, rb):
                assert np.array_equal(x, y)


def test_rel_err_metric():
    # bench.cpp:106-115 floor-1 metric
    assert oracle.rel_err([1e-9], [2e-9]) == pytest.approx(1e-9)
    assert oracle.rel_err([100.0], [101.0]) == pytest.approx(1 / 101)

"""CPU: the drop-in host API (C++ `graphfuse` namespace via the `_core`
pybind module) reproduces the reference's host-side behaviour exactly:
graph canonicalisation, seeded generators, planners, modelled counters,
error types and messages.  Expected values come from the reference itself
(tests/golden/, scripts/make_golden.py) and from the reference's own unit
tests (test_graph.cpp, test_schedule.cpp, test_engine.cpp).
"""
import os

import numpy as np
import pytest

import paper_2411_16127_b200 as gf
from paper_2411_16127_b200 import _core

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def graphs():
    return np.load(os.path.join(GOLD, "graphs.npz"))


def arrays(g):
    return {k: np.asarray(getattr(g, a), np.int64) for k, a in (
        ("row_ptr", "csr_row_ptr"), ("col", "csr_col_idx"), ("csc_ptr", "csc_col_ptr"),
        ("csc_row", "csc_row_idx"), ("csc_perm", "csc_edge_perm"))}


def check_graph(g, graphs, name):
    a = arrays(g)
    for k, v in a.items():
        assert np.array_equal(v, graphs[f"{name}/{k}"]), (name, k)


def test_from_coo(graphs):
    for name in ("coo3", "selfloops", "empty_rows", "rand40", "hub100", "citeseer"):
        n = int(graphs[f"{name}/n"])
        src, dst = graphs[f"{name}/src"], graphs[f"{name}/dst"]
        perm = np.random.default_rng(1).permutation(src.shape[0])
        check_graph(gf.from_coo(n, src[perm], dst[perm]), graphs, name)


def test_seeded_generators_reproduce_reference(graphs):
    check_graph(gf.gen_random(40, 4.0, 1), graphs, "rand40")
    check_graph(gf.gen_random(120, 5.0, 11), graphs, "rand120")
    check_graph(gf.gen_random(12, 3.0, 3), graphs, "rand12")
    check_graph(gf.gen_super_node(100, 4.0, 90, 7), graphs, "hub100")
    check_graph(gf.gen_random(3327, 9228.0 / 3327.0, 11), graphs, "citeseer")


def test_batch_graphs(graphs):
    g = gf.from_coo(3, np.array([0, 2, 1]), np.array([1, 1, 2]))
    b = gf.batch_graphs([g, g])
    assert list(b.csr_row_ptr) == list(graphs["batch2/row_ptr"])
    assert list(b.csr_col_idx) == list(graphs["batch2/col"])
    with pytest.raises(RuntimeError, match="empty list"):
        gf.batch_graphs([])


def test_graph_errors():
    with pytest.raises(RuntimeError, match="duplicate edge"):
        gf.from_coo(2, np.array([0, 0]), np.array([1, 1]))
    with pytest.raises(RuntimeError, match="out of range"):
        gf.from_coo(2, np.array([0]), np.array([2]))
    with pytest.raises(RuntimeError, match="avg_degree"):
        gf.gen_random(4, 4.0, 0)
    with pytest.raises(RuntimeError, match="hub_degree"):
        gf.gen_super_node(4, 1.0, 5, 0)


def test_degree_stats_and_threshold():
    star = gf.from_coo(6, np.array([1, 2, 3, 4, 5]), np.array([0, 0, 0, 0, 0]))
    avg, mx, mn = gf.degree_stats(star)
    assert mx == 5 and mn == 0 and avg == pytest.approx(5 / 6)
    assert gf.super_node_threshold(49152, 4) == 12288
    with pytest.raises(RuntimeError):
        gf.super_node_threshold(49152, 0)


def test_strategy_selection():
    # test_smoke.py:78-83 / test_schedule.cpp:9-26
    hub = gf.gen_super_node(100, 2.0, 90, 1)
    assert gf.select_strategy(hub, "dot", shared_mem_bytes=320, dtype_bytes=4) == "pmf"
    assert gf.select_strategy(hub, "add", shared_mem_bytes=320, dtype_bytes=4) == "smmf"
    assert gf.select_strategy(hub, "dot") == "smmf"
    with pytest.raises(ValueError):
        gf.select_strategy(hub, "mul")
    with pytest.raises(ValueError, match="unknown strategy"):
        _core.strategy_from_string("bogus")
    assert _core.strategy_from_string("feature-parallel") == "baseline"


def test_planners_known_answers():
    # test_schedule.cpp:44-121
    g = gf.from_coo(8, np.array([1, 2, 3, 4, 5, 6, 0, 0]), np.array([0, 0, 0, 0, 0, 0, 1, 2]))
    assert [e - b for b, e in _core.warp_balance(g, 0, 4, 4)] == [2, 2, 2, 2]
    g5 = gf.from_coo(5, np.array([0, 1, 2, 3, 4]), np.array([1, 1, 1, 2, 2]))
    assert [e - b for b, e in _core.warp_balance(g5, 0, 5, 4)] == [2, 1, 1, 1]
    g10 = gf.gen_random(10, 1, 2)
    assert [e - b for b, e in _core.edge_parallel_partition(g10, 3)] == [4, 3, 3]
    assert _core.edge_parallel_partition(gf.from_coo(3, np.array([]), np.array([])), 4) == []
    assert _core.partition_blocks(gf.gen_random(10, 0, 1), 4) == [(0, 4), (4, 8), (8, 10)]
    assert _core.shared_mem_usage(4, 4, 100, 64) == 1824
    with pytest.raises(ValueError):
        _core.partition_blocks(g10, 0)


def test_model_counters_match_reference(graphs):
    cz = np.load(os.path.join(GOLD, "counters.npz"))
    gen = {"rand120": lambda: gf.gen_random(120, 5.0, 11), "hub100": lambda: gf.gen_super_node(100, 4.0, 90, 7),
           "rand40": lambda: gf.gen_random(40, 4.0, 1)}
    keys = ["global_bytes_read", "global_bytes_written", "shared_bytes_accessed",
            "memory_transactions", "kernel_launches", "softmax_scalar_ops", "s_global_bytes",
            "f_global_bytes", "p_global_bytes", "max_group_load", "fallback_unfused"]
    strategies = ["smmf", "pmf", "unfused", "baseline"]
    names = sorted({k.split("/")[0] for k in cz.files})
    assert len(names) >= 9
    for name in names:
        d, var, l2, strat, rpb, groups, gw, vw, budget, db = (int(x) for x in cz[f"{name}/args"])
        g = gen[str(cz[f"{name}/graph"])]()
        c = _core.model_counters(g, "add" if var else "dot", d, strategies[strat], db, rpb,
                                 groups, gw, vw)
        got = [c[k] for k in keys]
        assert got == [int(x) for x in cz[f"{name}/counters"]], name
        assert list(c["per_group_edge_loads"]) == [int(x) for x in cz[f"{name}/loads"]], name


def test_smmf_feasibility_message():
    # test_engine.cpp:162-177: message names the block and what it requires
    g = gf.gen_super_node(100, 2.0, 90, 1)
    with pytest.raises(RuntimeError) as e:
        _core.check_smmf_feasible(g, 8, 256, 4)
    assert "block 0" in str(e.value) and "requires" in str(e.value)
    _core.check_smmf_feasible(g, 8, 1 << 20, 4)


def test_graph_io_roundtrip(tmp_path):
    g = gf.gen_random(30, 3.0, 77)
    p = str(tmp_path / "g.txt")
    gf.save_graph(p, g)
    r = gf.load_graph(p)
    assert list(r.csr_row_ptr) == list(g.csr_row_ptr)
    assert list(r.csr_col_idx) == list(g.csr_col_idx)
    with pytest.raises(RuntimeError, match="cannot open"):
        gf.load_graph(str(tmp_path / "missing.txt"))


def test_compute_entry_points_fail_loudly_without_gpu():
    """No CPU fallback: on a GPU-less host the compute API raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = gf.gen_random(10, 2.0, 1)
    x = np.zeros((10, 4))
    with pytest.raises(RuntimeError, match="no sm_100 device"):
        gf.forward(g, x, x, x)
    with pytest.raises(RuntimeError, match="no sm_100 device"):
        gf.backward(g, x, x, x, x)


def test_bench_config_errors_before_any_device_work():
    """run_benchmark_json (module.cpp:151-154) validates the config first: a
    missing peak_bw and malformed JSON raise BenchError -> RuntimeError
    (bench.cpp:51-53, 153-159), on a host with or without a GPU."""
    import json

    with pytest.raises(RuntimeError, match="peak_bw"):
        _core.run_benchmark_json(json.dumps({"model": "gt", "nodes": 50, "peak_bw": 0}))
    with pytest.raises(RuntimeError, match="bad config"):
        _core.run_benchmark_json("{ not json")
    with pytest.raises(RuntimeError, match="bad config"):
        _core.run_benchmark_json(json.dumps({"nodes": "many", "peak_bw": 1e12}))
    with pytest.raises(RuntimeError, match="unknown dtype"):
        _core.run_benchmark_json(json.dumps({"dtype": "f16", "peak_bw": 1e12}))

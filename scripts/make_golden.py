"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference sources).  Run here, where the reference
exists; the fixtures are committed and travel to the GPU box.

  python scripts/make_golden.py

Contents
  graphs.npz     reference from_coo / gen_random / gen_super_node / batch_graphs
                 outputs (CSR, CSC, csc_edge_perm) for fixed inputs / seeds
  pipeline.npz   multi-head forward (O, P) and backward (dQ, dK, dV) of the
                 reference (per-head run_strategy / fused_backward) on seeded
                 inputs, f32 and f64, GAT / GT / AGNN and generic shapes
  counters.npz   reference ExecCounters (modelled) for strategies x plans
"""
import os
import sys

import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

GRAPHS = {
    "coo3": ("coo", 3, [0, 2, 1], [1, 1, 2]),          # test_graph.cpp:11-22
    "selfloops": ("coo", 2, [0, 1], [0, 1]),             # test_graph.cpp:30-35
    "empty_rows": ("coo", 10, [0, 1], [7, 7]),           # test_engine.cpp:199-215
    "rand40": ("random", 40, 4.0, 1),                    # test_smoke.py small()
    "rand120": ("random", 120, 5.0, 11),
    "hub100": ("super", 100, 4.0, 90, 7),                # test_engine.cpp:97-120
    "rand12": ("random", 12, 3.0, 3),                    # test_smoke.py gradcheck
    "citeseer": ("random", 3327, 9228.0 / 3327.0, 11),   # test_graph.cpp degree stats
}

PIPE = [  # (name, graph, variant, l2, H, D, dtype)
    ("gat8x8_f32", "rand120", "add", False, 8, 8, np.float32),
    ("gt8x16_f32", "rand120", "dot", False, 8, 16, np.float32),
    ("agnn2x16_f32", "rand120", "dot", True, 2, 16, np.float32),
    ("gat8x8_f64", "rand120", "add", False, 8, 8, np.float64),
    ("gt2x5_f64", "rand120", "dot", False, 2, 5, np.float64),
    ("agnn1x6_f64", "rand40", "dot", True, 1, 6, np.float64),
    ("hub_gt4x8_f32", "hub100", "dot", False, 4, 8, np.float32),
    ("empty_dot1x4_f64", "empty_rows", "dot", False, 1, 4, np.float64),
]


def build_graph(spec):
    kind = spec[0]
    if kind == "coo":
        return oracle.ref_from_coo(spec[1], np.array(spec[2]), np.array(spec[3])), spec[2], spec[3]
    if kind == "random":
        g = oracle.ref_gen_random(*spec[1:])
    else:
        g = oracle.ref_gen_super_node(*spec[1:])
    a = g.arrays()
    return g, a.col, a.coo_dst


def main():
    os.makedirs(OUT, exist_ok=True)
    garr, refs = {}, {}
    for name, spec in GRAPHS.items():
        g, src, dst = build_graph(spec)
        a = g.arrays()
        refs[name] = g
        garr[f"{name}/n"] = np.array(a.n)
        garr[f"{name}/src"] = np.asarray(src, np.int64)
        garr[f"{name}/dst"] = np.asarray(dst, np.int64)
        for k in ("row_ptr", "col", "csc_ptr", "csc_row", "csc_perm"):
            garr[f"{name}/{k}"] = getattr(a, k)
    # batch_graphs({coo3, coo3}) -> test_graph.cpp:73-81
    c3 = refs["coo3"].arrays()
    s = np.concatenate([c3.col, c3.col + 3])
    d = np.concatenate([c3.coo_dst, c3.coo_dst + 3])
    b = oracle.ref_from_coo(6, s, d).arrays()
    garr["batch2/row_ptr"], garr["batch2/col"] = b.row_ptr, b.col
    np.savez_compressed(os.path.join(OUT, "graphs.npz"), **garr)

    parr = {}
    for name, gname, variant, l2, H, D, dt in PIPE:
        g = refs[gname]
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        w = H if variant == "add" else H * D
        amp = 2.0 if variant == "add" else 1.0
        Q = rng.uniform(-amp, amp, (g.n, w)).astype(dt)
        K = rng.uniform(-amp, amp, (g.n, w)).astype(dt)
        V = rng.uniform(-1, 1, (g.n, H * D)).astype(dt)
        dO = rng.uniform(-1, 1, (g.n, H * D)).astype(dt)
        scale = 1.0 / np.sqrt(D) if variant == "dot" and not l2 else 1.0
        O, P = oracle.ref_forward(g, Q, K, V, H, D, variant, l2, scale, 0.2, want_p=True)
        dQ, dK, dV = oracle.ref_backward(g, Q, K, V, dO, H, D, variant, l2, scale, 0.2)
        meta = np.array([H, D, int(variant == "add"), int(l2)], np.int64)
        for k, v in (("Q", Q), ("K", K), ("V", V), ("dO", dO), ("O", O), ("P", P), ("dQ", dQ),
                     ("dK", dK), ("dV", dV)):
            parr[f"{name}/{k}"] = v
        parr[f"{name}/meta"] = meta
        parr[f"{name}/scale"] = np.array(scale)
        parr[f"{name}/graph"] = np.array(gname)
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **parr)

    import ctypes as C

    carr = {}
    cases = [  # (name, graph, d, variant, l2, strategy, rpb, groups, gw, vw, budget, dtype_bytes)
        ("rand120_dot_smmf", "rand120", 8, 0, 0, 0, 4, 4, 32, 4, 1 << 20, 4),
        ("rand120_dot_pmf", "rand120", 8, 0, 0, 1, 4, 4, 32, 4, 1 << 20, 4),
        ("rand120_dot_unfused", "rand120", 8, 0, 0, 2, 4, 4, 32, 4, 1 << 20, 4),
        ("rand120_dot_base128", "rand120", 128, 0, 0, 3, 4, 4, 32, 4, 1 << 24, 4),
        ("rand120_add_smmf_f64", "rand120", 6, 1, 0, 0, 4, 4, 32, 4, 1 << 20, 8),
        ("hub100_dot_smmf", "hub100", 8, 0, 0, 0, 4, 4, 32, 4, 1 << 20, 4),
        ("hub100_dot_base", "hub100", 8, 0, 0, 3, 4, 4, 32, 4, 1 << 20, 4),
        ("rand40_vw1", "rand40", 64, 0, 0, 0, 4, 4, 32, 1, 1 << 22, 4),
        ("rand40_rpb3_g5", "rand40", 16, 0, 0, 0, 3, 5, 16, 2, 1 << 22, 8),
    ]
    for name, gname, d, var, l2, strat, rpb, groups, gw, vw, budget, db in cases:
        out = np.zeros(11, np.uint64)
        loads = np.zeros(100000, np.uint64)
        nl = np.zeros(1, np.int64)
        rc = oracle.ref().gfref_forward_counters(
            refs[gname].h, d, var, l2, strat, rpb, groups, gw, vw, budget, db,
            out.ctypes.data_as(C.c_void_p), loads.ctypes.data_as(C.c_void_p), loads.shape[0],
            nl.ctypes.data_as(C.c_void_p))
        assert rc == 0, oracle.ref().gfref_last_error()
        carr[f"{name}/counters"] = out
        carr[f"{name}/loads"] = loads[: nl[0]]
        carr[f"{name}/args"] = np.array([d, var, l2, strat, rpb, groups, gw, vw, budget, db],
                                        np.int64)
        carr[f"{name}/graph"] = np.array(gname)
    np.savez_compressed(os.path.join(OUT, "counters.npz"), **carr)

    # Layer level (models.hpp:104-158), single head, f64: conv_forward +
    # conv_backward of the reference on seeded X / weights / dO.
    conv = {}
    for mi, model in enumerate(("gt", "agnn", "gat")):
        g = refs["rand40"]
        rng = np.random.default_rng(100 + mi)
        d_in, dim = 5, 4
        X = rng.uniform(-1, 1, (g.n, d_in))
        lim = 1 / np.sqrt(d_in)
        Wq, Wk, Wv = (rng.uniform(-lim, lim, (d_in, dim)) for _ in range(3))
        al, ar = rng.uniform(-lim, lim, (dim, 1)), rng.uniform(-lim, lim, (dim, 1))
        dO = rng.uniform(-1, 1, (g.n, dim))
        O = np.zeros((g.n, dim))
        dWq, dWk, dWv = np.zeros((d_in, dim)), np.zeros((d_in, dim)), np.zeros((d_in, dim))
        dal, dar = np.zeros((dim, 1)), np.zeros((dim, 1))
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        rc = oracle.ref().gfref_conv_f64(g.h, mi, dim, d_in, 0.0, 0.2, P(X), P(Wq), P(Wk), P(Wv),
                                         P(al), P(ar), P(dO), P(O), P(dWq), P(dWk), P(dWv),
                                         P(dal), P(dar))
        assert rc == 0, oracle.ref().gfref_last_error()
        for k, v in (("X", X), ("Wq", Wq), ("Wk", Wk), ("Wv", Wv), ("al", al), ("ar", ar),
                     ("dO", dO), ("O", O), ("dWq", dWq), ("dWk", dWk), ("dWv", dWv),
                     ("dal", dal), ("dar", dar)):
            conv[f"{model}/{k}"] = v
    np.savez_compressed(os.path.join(OUT, "conv.npz"), **conv)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()

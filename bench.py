#!/usr/bin/env python
"""bench.py — fused AT-GNN layer fwd+bwd throughput on B200 (GEdges/s).

Metric (BASELINE.json): "fused AT-GNN layer fwd+bwd GEdges/s and % HBM
roofline, 1/2/4/8 B200 vs CPU".  One step = one fused forward (SDDMM ->
edge softmax -> SpMM, 1 launch) + the recompute backward (pass A over CSR
rows + pass B over CSC columns, 2 launches) of one GAT 8x8 fp32 layer over
the whole synthetic Reddit-shape power-law graph (BASELINE configs[3], C4:
N=232,965, E~114.4M, max in-degree 21,657), inputs resident in HBM.  Edges
are counted once per layer, all 8 heads included: value = E*K / sum(step).

Timing: CUDA events on the launching stream around every kernel, W untimed
warm-up steps, L2 flushed (256 MiB write) between timed steps (outside the
events), nvidia-smi clocks sampled during the timed region.  `e2e` is the
same metric through the C-ABI with pinned HOST buffers: the step's inputs are
copied H2D and its outputs D2H inside the timed region.  `cpu_baseline` is the
reference's own CPU implementation (oracle/_ref, compiled from the reference
sources) timed on this host on a bounded sample (one head, a row slice).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4|c1|c2|c3|c5gat|c5gt]

N>1 (torchrun): nodes are sharded into contiguous ranges balanced by in+out
edges (paper_2411_16127_b200/shard.py); each rank runs the three kernels on
its rows / columns and the step includes the NCCL all-gathers: V and Q|el
before the forward; dO (and K for dot models) issued on NCCL's stream under
the forward and pass A; the softmax records before pass B.  The graph is
fixed as N grows (strong scaling); value = all edges / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (graph, layer, H, D, description)
    "c1": ("cora", "gat", 8, 8, "C1 Cora-shape GAT 8x8 fp32 fwd+bwd"),
    "c2": ("molhiv", "gt", 8, 16, "C2 ogbg-molhiv-shape x1024 GT 8x16 fp32 fwd+bwd"),
    "c3": ("pubmed", "agnn", 1, 128, "C3 PubMed-shape AGNN 1x128 fp32 fwd+bwd"),
    "c4": ("reddit", "gat", 8, 8, "C4 Reddit-shape power-law GAT 8x8 fp32 fwd+bwd"),
    "c5gat": ("products", "gat", 8, 8, "C5 ogbn-products-shape GAT 8x8 fp32 fwd+bwd"),
    "c5gt": ("products", "gt", 8, 16, "C5 ogbn-products-shape GT 8x16 fp32 fwd+bwd"),
}
REDDIT_N, REDDIT_MAX, REDDIT_EXP = 232_965, 21_657, 0.34
L2_BYTES = 126 * 1024 * 1024


# ---------------------------------------------------------------- graphs --
def reddit_degrees(np):
    i = np.arange(REDDIT_N, dtype=np.float64)
    return np.rint(REDDIT_MAX * (i + 1.0) ** -REDDIT_EXP).astype(np.int64)


def gen_graph_device(name, device, seed=0):
    """Synthetic graph generated on the GPU by this package's device
    generators (gf_gen_*_device: counter-hashed draws + radix-sort dedup;
    setup only): returns (n, src, dst) int64 device tensors of distinct edges.
    The canonical CSR/CSC is then built by the device from_coo kernel,
    bit-exact with the reference's from_coo."""
    import numpy as np
    import torch

    from paper_2411_16127_b200 import fused

    if name == "reddit":
        # Chung-Lu-style in-degree sequence deg_i = round(21657 (i+1)^-0.34) on
        # hashed node ids, uniform sources, duplicate sources dropped
        src, dst = fused.gen_power_law_device(REDDIT_N, REDDIT_MAX, REDDIT_EXP, seed=seed,
                                              device=device)
        return REDDIT_N, src, dst
    if name in ("products", "pubmed", "cora"):
        n, e = {"products": (2_400_000, 62_000_000), "pubmed": (19_717, 88_648),
                "cora": (2_708, 10_556)}[name]
        src, dst = fused.gen_random_device(n, e / n, seed=seed, device=device)
        return n, src, dst
    if name == "molhiv":
        # 1024 molecules of 26 atoms: a random spanning tree + 3 ring bonds,
        # bonds in both directions (~25.5 atoms / 27.5 bonds per ogbg-molhiv graph).
        mols, atoms = 1024, 26
        src, dst = fused.gen_molecules_device(mols, atoms, 3, seed=seed, device=device)
        return mols * atoms, src, dst
    raise ValueError(name)


# ----------------------------------------------------------- measurement --
def algorithmic_bytes(kernel, layer, n, e, H, D, b=4, idx=4):
    """Per-launch algorithmic bytes (SURVEY §8(d) gather
    model with this design's stats layout): every gathered row counted per
    edge, every owned row once, index arrays once."""
    F = H * D
    dot = layer != "gat"
    qk = F if dot else H  # Q|el and K|er width
    rec = 4 * H  # softmax record {m, log2 l, aux, delta} per head
    topo = idx * (2 * n + 1 + e)  # row pointer, schedule, neighbour ids
    if kernel == "fwd":  # gather V, Q|el of src; own K|er; write O + records
        return topo + b * (e * (F + qk) + n * (qk + F + rec))
    if kernel == "bwd_rows":  # gather V, Q|el of src; own dO, O, K (dot), record; write dK|der, delta
        return topo + b * (e * (F + qk) + n * (2 * F + (F if dot else 0) + rec + qk + H))
    if kernel == "bwd_cols":  # gather dO, K (dot), record of dst; own V, Q|el; write dV, dQ|del
        return topo + b * (e * (F + (F if dot else 0) + rec) + n * (2 * F + 2 * qk))
    raise ValueError(kernel)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi has produced a sample (its start-up takes a
        few hundred ms), so the timed region is covered from its start."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.first = len(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows[max(0, getattr(self, "first", 1) - 1):]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def measured_l2_gather(row_bytes, footprint=64 << 20):
    """Live L2 gather peak (GB/s) for rows of the hot kernels' gathered row
    size from an L2-resident footprint (gf_measure_l2_gather; same 256-bit
    non-coherent loads).  The second roofline denominator: the C4 node tables
    (V 60 MB + el 7.5 MB) are L2-resident, so HBM is not the binding limit."""
    import ctypes as C

    from paper_2411_16127_b200._capi import check, lib

    rb = max(32, min(1024, (row_bytes + 31) // 32 * 32))
    g = C.c_double()
    check(lib().gf_measure_l2_gather(footprint, rb, 5, C.byref(g), None), "gf_measure_l2_gather")
    return g.value, rb


def l2_request_costs():
    """Per-request L2 gather costs (ps) fitted live from two probe points:
    a random 32 B row is one line + one sector, a 128 B row one line + four
    sectors (t = a*lines + b*sectors).  The 256 B point checks the fit."""
    g32, _ = measured_l2_gather(32)
    g128, _ = measured_l2_gather(128)
    t32, t128 = 32 / g32 * 1e3, 128 / g128 * 1e3  # ps per row
    b = (t128 - t32) / 3
    return t32 - b, b, g32, g128


def gathered_rows(kernel, layer, H, D, b=4):
    """Row sizes (bytes) each edge gathers in one launch."""
    F = H * D
    rec = 16 * H if b == 4 else 32 * H
    if layer == "gat":
        return {"fwd": [b * F, b * H], "bwd_rows": [b * F, b * H], "bwd_cols": [b * F, rec]}[kernel]
    return {"fwd": [b * F, b * F], "bwd_rows": [b * F, b * F],
            "bwd_cols": [b * F, b * F, rec]}[kernel]


def l2_request_model_ms(kernel, layer, H, D, e, a_ps, b_ps):
    """Modelled launch time when every gather is an L2 hit: per edge and
    gathered row, a line-request cost per 128 B line touched plus a sector
    cost per 32 B sector."""
    t = 0.0
    for rb in gathered_rows(kernel, layer, H, D):
        t += a_ps * max(1, -(-rb // 128)) + b_ps * max(1, -(-rb // 32))
    return e * t * 1e-9


def ncu_traffic(config, kernel):
    """DRAM bytes per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config, {}).get(kernel)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------- CPU baseline --
def row_slice_sample(n, row_ptr, col, frac):
    """Host CSR/CSC of the subgraph keeping the in-edges of the first rows
    (by id) that hold ~frac of the edges (ids are randomly permuted, so the
    slice has the graph's degree mix)."""
    import numpy as np

    e_total = int(row_ptr[-1])
    r = int(np.searchsorted(row_ptr, int(e_total * frac)))
    r = max(1, min(n, r))
    es = int(row_ptr[r])
    rp = np.concatenate([row_ptr[: r + 1], np.full(n - r, es, np.int64)]).astype(np.int64)
    c = np.ascontiguousarray(col[:es], np.int64)
    dst = np.repeat(np.arange(r, dtype=np.int64), np.diff(row_ptr[: r + 1]))
    order = np.argsort(c, kind="stable")
    csc_row = dst[order]
    csc_ptr = np.zeros(n + 1, np.int64)
    csc_ptr[1:] = np.cumsum(np.bincount(c, minlength=n))
    import oracle

    return oracle.CSR(n, rp, c, csc_ptr, csc_row, order.astype(np.int64))


def cpu_reference_sample(sub, layer, D, steps=1, seed=0):
    """Time the reference (oracle/_ref) on one head of the sampled subgraph:
    run_strategy<float> + fused_backward<float>.  Returns
    (GEdges/s for all H heads, seconds per head)."""
    import ctypes as C

    import numpy as np

    import oracle

    rg = oracle.ref_adopt(sub)
    rng = np.random.default_rng(seed)
    w = 1 if layer == "gat" else D
    q = rng.uniform(-1, 1, (sub.n, w)).astype(np.float32)
    k = rng.uniform(-1, 1, (sub.n, w)).astype(np.float32)
    v = rng.uniform(-1, 1, (sub.n, D)).astype(np.float32)
    do = rng.uniform(-1, 1, (sub.n, D)).astype(np.float32)
    variant = 1 if layer == "gat" else 0
    l2 = 1 if layer == "agnn" else 0
    scale = 1.0 if layer != "gt" else 1.0 / np.sqrt(D)
    times = []
    for _ in range(steps):
        f = C.c_double()
        b = C.c_double()
        rc = oracle.ref().gfref_time_head_f32(
            rg.h, D, variant, scale, 0.2, l2, q.ctypes.data_as(C.c_void_p),
            k.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
            do.ctypes.data_as(C.c_void_p), C.byref(f), C.byref(b))
        if rc:
            raise RuntimeError(oracle.ref().gfref_last_error().decode())
        times.append(f.value + b.value)
    return times, sub.e


# ----------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frac", type=float, default=0.5,
                    help="edge fraction of the CPU-baseline row slice")
    ap.add_argument("--cta-threshold", type=int, default=0)
    ap.add_argument("--no-layer", action="store_true",
                    help="skip the layer-level (projection + pipeline) measurement")
    ap.add_argument("--no-ablation", action="store_true",
                    help="skip the forward fusion-strategy ablation (smmf/pmf/unfused/baseline)")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="sharded training step: projected rows exchanged by the projection's own "
                         "epilogue into symmetric memory (p2p) or by NCCL all-gather")
    ap.add_argument("--phased", choices=("auto", "on", "off"), default="auto",
                    help="sharded step: source-phased forward overlapping the source-row exchange")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the row-sharded path (NCCL all-gathers) even at N=1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world)


# Edge fraction of the reference arm's per-step sample (a row slice; whole
# graph for the small configs) so one `--steps 50` run stays within minutes.
REF_SAMPLE_FRAC = {"cora": 1.0, "molhiv": 1.0, "pubmed": 1.0, "reddit": 1.0 / 16,
                   "products": 1.0 / 64}


def gen_graph_cpu(name, frac=1.0, seed=1):
    """The bench graphs' shapes generated on the CPU (numpy; the reference arm
    runs no GPU code), restricted to the destination rows [0, r) that hold
    ~frac of the edges (node ids are random, so the slice has the graph's
    degree mix).  Returns (n, src, dst) int64 unique edges."""
    import numpy as np

    rng = np.random.default_rng(seed)
    if name == "reddit":
        n = REDDIT_N
        deg_of = np.empty(n, np.int64)
        deg_of[rng.permutation(n)] = reddit_degrees(np)
        cum = np.cumsum(deg_of)
        r = int(np.searchsorted(cum, cum[-1] * frac)) + 1
        dst = np.repeat(np.arange(r, dtype=np.int64), deg_of[:r])
        src = rng.integers(0, n, dst.shape[0])
    elif name == "molhiv":
        mols, atoms = 1024, 26
        s_all, d_all = [], []
        for m in range(mols):
            base = m * atoms
            parent = [rng.integers(0, i) for i in range(1, atoms)]
            a = [base + i for i in range(1, atoms)] + [base + x for x in rng.integers(0, atoms, 3)]
            b = [base + p for p in parent] + [base + x for x in rng.integers(0, atoms, 3)]
            s_all += a + b
            d_all += b + a
        n = mols * atoms
        src, dst = np.array(s_all, np.int64), np.array(d_all, np.int64)
        keep = src != dst
        src, dst = src[keep], dst[keep]
    else:
        n, e = {"cora": (2_708, 10_556), "pubmed": (19_717, 88_648),
                "products": (2_400_000, 62_000_000)}[name]
        r = max(1, int(round(n * frac)))
        e_s = int(round(e * r / n))
        src = rng.integers(0, n, e_s)
        dst = rng.integers(0, r, e_s)
    key = np.unique(dst * n + src)
    return n, key % n, key // n


def run_reference(args, rank, world):
    """The reference's own CPU path (oracle/_ref), rank 0 only, on a bounded
    sample of the same workload per step."""
    import numpy as np

    graph, layer, H, D, desc = CONFIGS[args.config]
    if rank != 0:
        return 0
    import oracle

    frac = REF_SAMPLE_FRAC[graph]
    n, src, dst = gen_graph_cpu(graph, frac)
    sub = oracle.from_coo(n, src, dst)
    times, es = cpu_reference_sample(sub, layer, D, steps=args.warmup + args.steps)
    t = times[args.warmup:]
    per_step = sum(t) / len(t) * H  # one call per head, H heads
    value = es / per_step / 1e9
    out = {
        "metric": "fused AT-GNN layer fwd+bwd GEdges/s", "value": value, "unit": "GEdges/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "sample_edges": es,
                   "sample": f"1 head x row slice ({frac:g} of the edges), x{H} heads"},
        "cpu_baseline": {"value": value, "unit": "GEdges/s", "cores": os.cpu_count(),
                         "kind": "reference",
                         "sample": f"reference run_strategy<float>+fused_backward<float>, 1 of {H} "
                                   f"heads on a {es}-edge row slice ({frac:g} of E) of a CPU-generated "
                                   f"{graph}-shape graph; fwd uses all hardware threads, bwd is "
                                   "single-threaded by construction"},
        "e2e": {"value": value, "unit": "GEdges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def gat_layer(layer):
    return layer == "gat"


def layer_step_timing(args, layer, spec, dg, n, e, F, H, D, dev, stream, flush, shard=None):
    """One full-graph training step of the layer, fp32 (models.hpp:104-158 +
    an SGD update): projection of the owned rows (tcgen05 3xTF32), GAT
    logits, [sharded: all-gather of the projected source rows], fused
    attention forward + recompute backward, GAT fan-in, weight gradients
    X^T dY over the owned rows (tcgen05), [sharded: all-reduce of dW], SGD
    update of every weight.  X has width F (bench.cpp:86-87)."""
    import torch

    from paper_2411_16127_b200 import fused

    g = torch.Generator(device=dev)
    g.manual_seed(77)
    lim = 1.0 / F ** 0.5
    X = torch.rand(n, F, device=dev, generator=g) * 2 - 1
    dO = torch.rand(n, F, device=dev, generator=g) * 2 - 1
    rnd = lambda *s: (torch.rand(*s, device=dev, generator=g) * 2 - 1) * lim  # noqa: E731
    gat = layer == "gat"
    lr = 1e-3
    Wv = rnd(F, F)
    if gat:
        al, ar = rnd(F), rnd(F)
    else:
        Wq, Wk = rnd(F, F), rnd(F, F)
    rows = shard.block if shard is not None else slice(0, n)
    # Sharded exchange of the projected rows: "p2p" = the projection's
    # epilogue writes every rank's copy of the tables (gf_gemm_bcast into
    # symmetric memory, device barrier); "nccl" = projection, then all-gather.
    pt, exchange = None, None
    if shard is not None:
        exchange = "nccl"
        if getattr(args, "exchange", "p2p") == "p2p":
            try:
                from paper_2411_16127_b200.shard import PeerTables

                pt = PeerTables(shard, {"V": F} if gat_layer(layer) else {"Q": F, "K": F, "V": F},
                                device=dev)
                pt.selftest()
                exchange = "p2p: gemm_bcast epilogue into symmetric-memory tables + device barrier"
            except Exception as ex:  # recorded in the JSON line, NCCL path used
                exchange = f"nccl (p2p unavailable: {type(ex).__name__}: {str(ex)[:120]})"
    Hf = pt.table("V") if pt is not None else torch.zeros(n, F, device=dev)
    Qb = pt.table("Q") if pt is not None and not gat_layer(layer) else torch.zeros(n, F, device=dev)
    Kb = pt.table("K") if pt is not None and not gat_layer(layer) else torch.zeros(n, F, device=dev)
    EL = torch.zeros(n, H, device=dev)
    ER = torch.zeros(n, H, device=dev)
    O = torch.empty(n, F, device=dev)
    st = torch.zeros(n, H, 4, device=dev)
    qk = spec.qk_width
    dQ, dK, dV = (torch.zeros(n, qk, device=dev), torch.zeros(n, qk, device=dev),
                  torch.zeros(n, F, device=dev))
    dW = [torch.empty(F, F, device=dev) for _ in range(3)]
    Xr = X[rows]
    if shard is not None:
        import torch.distributed as dist

        from paper_2411_16127_b200.shard import all_gather_rows

    def step(ev=None):
        rec = (lambda i: ev[i].record(stream)) if ev else (lambda i: None)
        rec(0)
        later = []
        if pt is not None:
            pt.barrier()  # every rank is done reading the previous step's tables
            if gat:
                fused.gemm_bcast(Xr, Wv, pt.dests("V"), stream=stream)
                pt.barrier()
                # el / er of every row from the complete table (deterministic per
                # row, so identical to the owners' values): no logit exchange
                fused.gat_logits(Hf, al, ar, H, D, stream=stream, el=EL, er=ER)
                q, k, v = EL, ER, Hf
            else:
                for w_, name in ((Wq, "Q"), (Wk, "K"), (Wv, "V")):
                    fused.gemm_bcast(Xr, w_, pt.dests(name), stream=stream)
                pt.barrier()
                q, k, v = Qb, Kb, Hf
            later = [all_gather_rows(dO, shard, async_op=True)]
        elif gat:
            fused.gemm(Xr, Wv, out=Hf[rows], stream=stream)
            fused.gat_logits(Hf[rows], al, ar, H, D, stream=stream, el=EL[rows], er=ER[rows])
            q, k, v = EL, ER, Hf
        else:
            fused.gemm(Xr, Wq, out=Qb[rows], stream=stream)
            fused.gemm(Xr, Wk, out=Kb[rows], stream=stream)
            fused.gemm(Xr, Wv, out=Hf[rows], stream=stream)
            q, k, v = Qb, Kb, Hf
        if shard is not None and pt is None:  # source rows first; dO (and K) under fwd / pass A
            for w in [all_gather_rows(t, shard, async_op=True) for t in (v, q)]:
                w.wait()
            later = [all_gather_rows(t, shard, async_op=True)
                     for t in (dO,) + (() if gat else (k,))]
        rec(1)
        fused.attn_forward(dg, spec, q, k, v, O=O, stats=st, stream=stream)
        fused.attn_backward_rows(dg, spec, q, k, v, O, st, dO, dK, stream=stream)
        if shard is not None:
            for w in later:
                w.wait()
            all_gather_rows(st, shard)
        fused.attn_backward_cols(dg, spec, q, k, v, st, dO, dQ, dV, stream=stream)
        rec(2)
        if gat:
            dH, dal, dar = fused.gat_fanin(Hf[rows], al, ar, dV[rows], dQ[rows], dK[rows], H, D,
                                           stream=stream)
            fused.gemm(Xr, dH, trans_a=True, out=dW[0], stream=stream)
            grads = [(Wv, dW[0]), (al, dal), (ar, dar)]
        else:
            for w_, d_ in zip(dW, (dQ, dK, dV)):
                fused.gemm(Xr, d_[rows], trans_a=True, out=w_, stream=stream)
            grads = [(Wq, dW[0]), (Wk, dW[1]), (Wv, dW[2])]
        if shard is not None:  # weight gradients are partial sums over the owned rows
            for _, d_ in grads:
                dist.all_reduce(d_)
        rec(3)
        for w_, d_ in grads:  # SGD
            w_.add_(d_, alpha=-lr)
        rec(4)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = max(5, args.steps // 5)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    if shard is not None:
        dist.barrier()
    for i in range(K):
        flush.zero_()
        step(evs[i])
    torch.cuda.synchronize()
    seg = lambda j: sum(a[j].elapsed_time(a[j + 1]) for a in evs) / K  # noqa: E731
    ms = sum(a[0].elapsed_time(a[4]) for a in evs) / K
    if shard is not None:  # whole job: max over ranks
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": e / (ms / 1e3) / 1e9, "unit": "GEdges/s", "ms_per_step": ms,
            "projection_fwd_ms": seg(0), "pipeline_ms": seg(1), "weight_grad_ms": seg(2),
            "sgd_ms": seg(3),
            "step": "projection (+ all-gather when sharded) -> fused attention fwd + recompute "
                    "bwd -> GAT fan-in -> X^T dY (+ all-reduce when sharded) -> SGD update",
            "projection": "X*W and X^T*dY on tcgen05 (3xTF32, UTCHMMA; X^T*dY deterministic split-K)",
            "exchange": exchange,
            "x_width": F}


def strategy_ablation(dg, spec, Q, K, V, O, stats, stream, flush, steps=5):
    """Forward time per fusion strategy (the paper's ablation, DF-GNN §5):
    SMMF (this design's default), PMF, unfused and the feature-parallel
    baseline, each on the same inputs with L2 flushed before every launch
    group; CUDA events on the launching stream."""
    import torch

    from paper_2411_16127_b200 import fused

    out = {}
    for strat in ("smmf", "pmf", "unfused", "baseline"):
        try:
            ws = fused.strategy_workspace(dg, spec, strat, dtype=V.dtype, device=V.device)
            for _ in range(2):
                fused.attn_forward(dg, spec, Q, K, V, O=O, stats=stats, stream=stream,
                                   strategy=strat, workspace=ws)
            ms = []
            for _ in range(steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fused.attn_forward(dg, spec, Q, K, V, O=O, stats=stats, stream=stream,
                                   strategy=strat, workspace=ws)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            out[strat] = round(statistics.mean(ms), 4)
            del ws
        except Exception as ex:  # reported, never silently replaced
            out[strat] = f"failed: {ex}"
    torch.cuda.synchronize()
    return out


def backward_ablation(dg, spec, Q, K, V, O, stats, dO, stream, flush, steps=5):
    """Backward time: this design's fused recompute (pass A + pass B, nothing
    E x H in HBM) vs the reference's unfused 5-launch schedule (dP + dV,
    softmax backward, dQ + dK over a stored P, autograd.hpp:158-170)."""
    import torch

    from paper_2411_16127_b200 import fused

    out = {}
    try:
        O, stats, P = fused.attn_forward(dg, spec, Q, K, V, want_p=True, stream=stream)
        runs = {"fused": lambda: fused.attn_backward(dg, spec, Q, K, V, O, stats, dO, stream=stream),
                "unfused": lambda: fused.attn_backward_unfused(dg, spec, Q, K, V, P, dO,
                                                               stream=stream)}
        for name, fn in runs.items():
            for _ in range(2):
                fn()
            ms = []
            for _ in range(steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            out[name] = round(statistics.mean(ms), 4)
        del P
    except Exception as ex:  # reported, never silently replaced
        out["error"] = str(ex)
    torch.cuda.synchronize()
    return out


def e2e_pipelined(dg, spec, tabs, stream, steps, warmup=2):
    """End-to-end throughput through the C-ABI with HOST buffers, steps
    pipelined over two buffer sets: every step copies ITS OWN inputs (Q|el,
    K|er, V, dO) host->device and its outputs (O, dQ|del, dK|der, dV)
    device->host inside the timed region, and step i+1's upload and step
    i-1's download run on copy streams under step i's kernels (the serving
    arrangement for independent requests).  Returns ms per step."""
    import torch

    from paper_2411_16127_b200 import fused

    ins, outs = ("Q", "K", "V", "dO"), ("O", "dQ", "dK", "dV")
    sets = []
    for b in range(2):
        d = {k: torch.empty_like(v) for k, v in tabs.items()}
        hi = {k: tabs[k].cpu().pin_memory() for k in ins}
        ho = {k: torch.empty(tabs[k].shape, dtype=tabs[k].dtype).pin_memory() for k in outs}
        sets.append((d, hi, ho))
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    comp_done, out_done = [None, None], [None, None]

    def step(i):
        b = i % 2
        d, hi, ho = sets[b]
        if comp_done[b] is not None:  # step i-2 has finished reading inputs b
            s_in.wait_event(comp_done[b])
        with torch.cuda.stream(s_in):
            for k in ins:
                d[k].copy_(hi[k], non_blocking=True)
        ev_in = torch.cuda.Event()
        ev_in.record(s_in)
        stream.wait_event(ev_in)
        if out_done[b] is not None:  # step i-2's outputs b are on the host
            stream.wait_event(out_done[b])
        fused.attn_forward(dg, spec, d["Q"], d["K"], d["V"], O=d["O"], stats=d["stats"],
                           stream=stream)
        ev_f = torch.cuda.Event()
        ev_f.record(stream)
        fused.attn_backward_rows(dg, spec, d["Q"], d["K"], d["V"], d["O"], d["stats"], d["dO"],
                                 d["dK"], stream=stream)
        fused.attn_backward_cols(dg, spec, d["Q"], d["K"], d["V"], d["stats"], d["dO"], d["dQ"],
                                 d["dV"], stream=stream)
        ev_c = torch.cuda.Event()
        ev_c.record(stream)
        comp_done[b] = ev_c
        s_out.wait_event(ev_f)
        with torch.cuda.stream(s_out):
            ho["O"].copy_(d["O"], non_blocking=True)
        s_out.wait_event(ev_c)
        with torch.cuda.stream(s_out):
            for k in ("dQ", "dK", "dV"):
                ho[k].copy_(d[k], non_blocking=True)
        ev_o = torch.cuda.Event()
        ev_o.record(s_out)
        out_done[b] = ev_o

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    s_in.wait_event(start)
    s_out.wait_event(start)
    for i in range(steps):
        step(warmup + i)
    for ev in out_done:
        stream.wait_event(ev)
    end.record(stream)
    end.synchronize()
    return start.elapsed_time(end) / steps


def e2e_graphed(dg, spec, tabs, hin, hout, flush, steps):
    """The serial end-to-end step (H2D of Q|el, K|er, V, dO from pinned host
    memory -> forward -> pass A -> pass B -> D2H of O, dQ|del, dK|der, dV)
    captured once into a CUDA graph and replayed: one launch per step instead
    of eleven API calls, which is what bounds the small graphs (C1-C3).
    L2 flushed between replays.  Returns {"ms": ...} or {"error": ...}."""
    import torch

    from paper_2411_16127_b200 import fused

    Q, K, V, dO = (tabs[k] for k in ("Q", "K", "V", "dO"))
    O, st, dQ, dK, dV = (tabs[k] for k in ("O", "stats", "dQ", "dK", "dV"))

    def body():
        cs = torch.cuda.current_stream()
        for h, d in zip(hin, (Q, K, V, dO)):
            d.copy_(h, non_blocking=True)
        fused.attn_forward(dg, spec, Q, K, V, O=O, stats=st, stream=cs)
        fused.attn_backward_rows(dg, spec, Q, K, V, O, st, dO, dK, stream=cs)
        fused.attn_backward_cols(dg, spec, Q, K, V, st, dO, dQ, dV, stream=cs)
        for h, d in zip(hout, (O, dQ, dK, dV)):
            h.copy_(d, non_blocking=True)

    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()  # warm-up outside the capture
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        del g
        return {"ms": statistics.mean(ts)}
    except Exception as ex:  # reported, the other e2e numbers stand
        torch.cuda.synchronize()
        return {"error": f"{type(ex).__name__}: {str(ex)[:160]}"}


def run_ours(args, rank, world):
    import numpy as np
    import torch

    from paper_2411_16127_b200 import fused

    graph, layer, H, D, desc = CONFIGS[args.config]
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.force_shard
    if sharded:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    # ---- graph (setup, untimed): device generator -> device from_coo -> schedules
    n, src, dst = gen_graph_device(graph, dev)
    torch.cuda.synchronize()
    t_pre = time.perf_counter()
    row_ptr, col, csc_ptr, csc_row, _ = fused.from_coo_device(n, src, dst)
    torch.cuda.synchronize()
    pre_coo_ms = (time.perf_counter() - t_pre) * 1e3
    del src, dst
    e = int(col.numel())
    spec = fused.AttnSpec("add" if layer == "gat" else "dot", H, D,
                          scale=(1.0 / np.sqrt(D)) if layer == "gt" else 1.0, slope=0.2,
                          l2=layer == "agnn")
    F = H * D
    qk = spec.qk_width
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)  # every rank draws the same global tables

    def u(*shape, amp=1.0):
        return (torch.rand(*shape, device=dev, generator=gen) * 2 - 1) * amp

    amp = 2.0 if layer == "gat" else 1.0
    Q, K, V, dO = u(n, qk, amp=amp), u(n, qk, amp=amp), u(n, F), u(n, F)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream()
    shard = None
    if sharded:
        # Row-sharded (paper_2411_16127_b200/shard.py): padded id space, this
        # rank's block of every node table is its own nodes' rows.
        from paper_2411_16127_b200.shard import RowShard, all_gather_rows

        shard = RowShard.build(n, row_ptr, col, csc_ptr, csc_row, rank, world)
        dg = shard.device_graph(cta_threshold=args.cta_threshold)
        Q, K, V, dO = (shard.to_padded(x) for x in (Q, K, V, dO))
        n_tab = shard.n_padded
    else:
        t_pre = time.perf_counter()
        dg = fused.DeviceGraph.from_device_csr(n, row_ptr, col, csc_ptr, csc_row,
                                               cta_threshold=args.cta_threshold)
        torch.cuda.synchronize()
        pre_sched_ms = (time.perf_counter() - t_pre) * 1e3
        n_tab = n
    need_cpu = rank == 0 and not sharded and not args.no_cpu_baseline
    host_rp = row_ptr.cpu().numpy() if need_cpu else None
    host_col = col.cpu().numpy() if need_cpu else None
    del row_ptr, col, csc_ptr, csc_row
    O = torch.zeros(n_tab, F, device=dev)
    stats = torch.zeros(n_tab, H, 4, device=dev)
    dQ, dK, dV = (torch.zeros(n_tab, qk, device=dev), torch.zeros(n_tab, qk, device=dev),
                  torch.zeros(n_tab, F, device=dev))
    NEV = 6 if sharded else 4
    # Source-phased forward (shard.py): the source rows arrive per block
    # (broadcast from each owner) while the forward runs block by block, own
    # block first, then the partials are merged.  "auto": when the modelled
    # exposed exchange (the V, Q|el blocks of the other ranks at ~700 GB/s)
    # exceeds twice the phases' extra cost (partial O / records written and
    # merged, one launch per block).
    phased = False
    if sharded:
        from paper_2411_16127_b200 import shard as shard_mod

        row_b = 4 * (F + qk)
        ag_ms = (world - 1) / world * n_tab * row_b / 700e9 * 1e3
        # partials written, read back and merged (measured at N = 1: C5 GT +1.1 ms)
        extra_ms = world * shard.R * (F + 4 * H) * 4 * 3 / 5e12 * 1e3 + world * 0.02
        phased = args.phased == "on" or (args.phased == "auto" and ag_ms > 2 * extra_ms)
        if phased:
            parts = shard_mod.source_parts(shard, cta_threshold=args.cta_threshold)
            O_parts, rec_parts = shard_mod.part_buffers(parts, spec, device=dev)
            order = shard_mod.phase_order(shard)

    def step(ev=None):
        rec = (lambda i: ev[i].record(stream)) if ev else (lambda i: None)
        k = 0
        rec(k)
        later = []
        if sharded and phased:
            R = shard.R
            blocks = {b: [torch.distributed.broadcast(t[b * R:(b + 1) * R], src=b, async_op=True)
                          for t in (V, Q)] for b in range(world)}
            later = [all_gather_rows(t, shard, async_op=True)
                     for t in (dO,) + ((K,) if layer != "gat" else ())]
            k += 1
            rec(k)
            for b in order:  # own block first: its rows are already local
                if b != rank:
                    for w in blocks[b]:
                        w.wait()
                shard_mod.phase_forward(parts, b, spec, Q, K, V, O_parts, rec_parts,
                                        stream=stream)
            shard_mod.merge_phases(parts, spec, O_parts, rec_parts, O, stats, stream=stream)
        elif sharded:
            # exchange 1: source-side rows the forward gathers (V, Q|el) — waited
            # on; then dO and, for dot models, K (only pass B gathers them) are
            # issued on NCCL's stream and overlap the forward and pass A
            first = [all_gather_rows(t, shard, async_op=True) for t in (V, Q)]
            later = [all_gather_rows(t, shard, async_op=True)
                     for t in (dO,) + ((K,) if layer != "gat" else ())]
            for w in first:
                w.wait()
            k += 1
            rec(k)
        if not phased:
            fused.attn_forward(dg, spec, Q, K, V, O=O, stats=stats, stream=stream)
        k += 1
        rec(k)
        fused.attn_backward_rows(dg, spec, Q, K, V, O, stats, dO, dK, stream=stream)
        k += 1
        rec(k)
        if sharded:  # exchange 2: the softmax records (complete only after pass A)
            for w in later:
                w.wait()
            all_gather_rows(stats, shard)
            k += 1
            rec(k)
        fused.attn_backward_cols(dg, spec, Q, K, V, stats, dO, dQ, dV, stream=stream)
        k += 1
        rec(k)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(NEV)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        clk.wait_first()
        if sharded:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            step(evs[i])
        torch.cuda.synchronize()
        if sharded:
            torch.distributed.barrier()
        torch.cuda.synchronize()
    seg = [[a[j].elapsed_time(a[j + 1]) for a in evs] for j in range(NEV - 1)]
    if sharded:
        k_ag1, k_fwd, k_ra, k_ag2, k_rb = seg
    else:
        k_fwd, k_ra, k_rb = seg
        k_ag1 = k_ag2 = [0.0]
    tot = [evs[i][0].elapsed_time(evs[i][NEV - 1]) for i in range(args.steps)]
    sum_ms = sum(tot)
    if sharded:
        t = torch.tensor([sum_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        sum_ms = float(t.item())
    ms_per_step = sum_ms / args.steps
    value = e * args.steps / (sum_ms / 1e3) / 1e9

    # ---- e2e through the C-ABI with pinned host buffers
    e2e_val, e2e_serial, h2d, d2h, e2e_graph = None, None, 0, 0, None
    if not sharded:
        hQ, hK, hV, hdO = [x.cpu().pin_memory() for x in (Q, K, V, dO)]
        hO, hdQ, hdK, hdV = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (O, dQ, dK, dV)]
        h2d = sum(x.numel() * x.element_size() for x in (hQ, hK, hV, hdO))
        d2h = sum(x.numel() * x.element_size() for x in (hO, hdQ, hdK, hdV))

        # Copies overlap compute WITHIN the step (each step still moves all of
        # its own inputs H2D and outputs D2H): dO's H2D runs under the forward,
        # O's D2H under the backward, dK's D2H under pass B.
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_step():
            ev_start = torch.cuda.Event()
            ev_start.record(stream)
            for h, d in ((hQ, Q), (hK, K), (hV, V)):
                d.copy_(h, non_blocking=True)
            s_in.wait_event(ev_start)
            with torch.cuda.stream(s_in):
                dO.copy_(hdO, non_blocking=True)
            ev_do = torch.cuda.Event()
            ev_do.record(s_in)
            fused.attn_forward(dg, spec, Q, K, V, O=O, stats=stats, stream=stream)
            ev_f = torch.cuda.Event()
            ev_f.record(stream)
            s_out.wait_event(ev_f)
            with torch.cuda.stream(s_out):
                hO.copy_(O, non_blocking=True)
            stream.wait_event(ev_do)
            fused.attn_backward_rows(dg, spec, Q, K, V, O, stats, dO, dK, stream=stream)
            ev_a = torch.cuda.Event()
            ev_a.record(stream)
            s_out.wait_event(ev_a)
            with torch.cuda.stream(s_out):
                hdK.copy_(dK, non_blocking=True)
            fused.attn_backward_cols(dg, spec, Q, K, V, stats, dO, dQ, dV, stream=stream)
            for h, d in ((hdQ, dQ), (hdV, dV)):
                h.copy_(d, non_blocking=True)
            ev_o = torch.cuda.Event()
            ev_o.record(s_out)
            stream.wait_event(ev_o)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        ee = []
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            b.synchronize()
            ee.append(a.elapsed_time(b))
        e2e_serial = e / (statistics.mean(ee) / 1e3) / 1e9
        tabs = {"Q": Q, "K": K, "V": V, "dO": dO, "O": O, "stats": stats, "dQ": dQ, "dK": dK,
                "dV": dV}
        e2e_ms = e2e_pipelined(dg, spec, tabs, stream, args.steps)
        e2e_val = e / (e2e_ms / 1e3) / 1e9
        e2e_graph = e2e_graphed(dg, spec, tabs, (hQ, hK, hV, hdO), (hO, hdQ, hdK, hdV), flush,
                                max(3, args.steps // 2))
        if e2e_graph.get("ms"):
            e2e_graph["value"] = e / (e2e_graph["ms"] / 1e3) / 1e9
    else:
        # Row-sharded: every rank uploads ITS OWN rows of Q|el, K|er, V, dO from
        # pinned host memory, runs the step (NCCL all-gathers included) and
        # downloads its own rows of O, dQ|del, dK|der, dV; max over ranks.
        own = shard.rows
        hin = [x[own].cpu().pin_memory() for x in (Q, K, V, dO)]
        hout = [torch.empty(x[own].shape, dtype=x.dtype).pin_memory() for x in (O, dQ, dK, dV)]
        h2d = sum(x.numel() * x.element_size() for x in hin)
        d2h = sum(x.numel() * x.element_size() for x in hout)

        def e2e_step():
            for h, d in zip(hin, (Q, K, V, dO)):
                d[own].copy_(h, non_blocking=True)
            step()
            for h, d in zip(hout, (O, dQ, dK, dV)):
                h.copy_(d[own], non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(3, args.steps // 2)
        a.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        b.record(stream)
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_serial = e * n_e2e / (float(t.item()) / 1e3) / 1e9
        e2e_val = e2e_serial

    # ---- layer level (projections reported separately): the
    # conv_forward / conv_backward step of models.hpp:104-158 with X of width
    # F (bench.cpp:86-87): X·W on tcgen05 (3xTF32), GAT logits / fan-in,
    # the fused pipeline, and the weight gradients X^T·dH.
    layer_out = None
    if not args.no_layer:
        layer_out = layer_step_timing(args, layer, spec, dg, n_tab, e, F, H, D, dev, stream, flush,
                                      shard=shard)
    ablation = bwd_ablation = None
    if not sharded and not args.no_ablation:
        ablation = strategy_ablation(dg, spec, Q, K, V, O, stats, stream, flush)
        bwd_ablation = backward_ablation(dg, spec, Q, K, V, O, stats, dO, stream, flush)

    # ---- roofline of the dominant kernel
    means = {"fwd": statistics.mean(k_fwd), "bwd_rows": statistics.mean(k_ra),
             "bwd_cols": statistics.mean(k_rb)}
    dom = max(means, key=means.get)
    # per-launch algorithmic bytes of THIS rank's launches (owned nodes / edges)
    nb = (shard.hi - shard.lo) if sharded else n
    e_of = {"fwd": dg.e, "bwd_rows": dg.e,
            "bwd_cols": int(shard.csc_row.numel()) if sharded else dg.e}
    ab = algorithmic_bytes(dom, layer, nb, e_of[dom], H, D)
    achieved = ab / (means[dom] / 1e3) / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic = ncu_traffic(args.config, dom)
    step_bytes = sum(algorithmic_bytes(k, layer, nb, e_of[k], H, D) for k in means)
    l2_peak, l2_rb = measured_l2_gather(F * 4)
    a_ps, b_ps, g32, g128 = l2_request_costs()
    req_model = {k: l2_request_model_ms(k, layer, H, D, e_of[k], a_ps, b_ps) for k in means}
    # node tables the dominant kernel gathers (fwd / pass A: V and Q|el; pass B:
    # dO, K (dot) and the records): the L2 denominator applies when they fit L2
    gathered = {"fwd": F + qk, "bwd_rows": F + qk,
                "bwd_cols": F + (F if layer != "gat" else 0) + 4 * H}
    tables_bytes = 4 * n * gathered[dom]

    cpu = None
    if need_cpu:
        try:
            t0 = time.time()
            sub = row_slice_sample(n, host_rp, host_col, args.cpu_frac)
            times, es = cpu_reference_sample(sub, layer, D, steps=1)
            cpu_v = es / (times[0] * H) / 1e9
            cpu = {"value": cpu_v, "unit": "GEdges/s", "cores": os.cpu_count(),
                   "kind": "reference",
                   "sample": f"reference (oracle/_ref) run_strategy<float>+fused_backward<float>, "
                             f"1 of {H} heads on a {es}-edge row slice ({args.cpu_frac:g} of E) "
                             f"of the same graph, x{H} heads; fwd uses all hardware threads, "
                             f"bwd is single-threaded by construction; {time.time() - t0:.1f}s"}
        except Exception as ex:  # reported, never silently replaced
            cpu = {"value": None, "unit": "GEdges/s", "cores": os.cpu_count(),
                   "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        info = dg.info
        out = {
            "metric": "fused AT-GNN layer fwd+bwd GEdges/s", "value": value, "unit": "GEdges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "nodes": n, "edges": e, "heads": H, "head_dim": D,
                       "max_in_degree": int(info.max_in_degree),
                       "cta_rows": int(info.n_cta_rows), "cta_threshold": int(info.cta_threshold),
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"row-sharded x{world} (NCCL all-gather)" if sharded else "1 GPU"},
            "kernels_ms": {k: round(v, 4) for k, v in means.items()},
            "preprocess_ms": ({"from_coo": round(pre_coo_ms, 2), "schedule": round(pre_sched_ms, 2),
                               "note": "one-time graph setup on the device, wall clock with syncs: "
                                       "COO -> validated, deduplicated CSR + CSC + edge permutation "
                                       "(graph.cpp:25-78), then degree stats, buckets and "
                                       "schedules; the reference's CPU from_coo is 16.9 s on C4 "
                                       "(SURVEY a2)"} if not sharded else None),
            "phased_forward": phased if sharded else None,
            "allgather_ms": ({"src_rows_exposed": round(statistics.mean(k_ag1), 4),
                              "dO_K_records_exposed": round(statistics.mean(k_ag2), 4),
                              "note": "exposed on the compute stream: dO (and K for dot "
                                      "models) are all-gathered under the forward and pass A"}
                             if sharded else None),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "algorithmic_bytes": ab},
            "l2_roofline": {"bound": "l2", "kernel": dom, "achieved": achieved, "peak": l2_peak,
                            "applies": tables_bytes <= L2_BYTES,
                            "gathered_tables_bytes": tables_bytes,
                            "unit": "GB/s", "frac": achieved / l2_peak,
                            "step_frac": step_bytes / (ms_per_step / 1e3) / 1e9 / l2_peak,
                            "peak_kind": f"measured live: gf_measure_l2_gather, {l2_rb} B rows "
                                         "(the gathered row size), 64 MiB L2-resident footprint"},
            "l2_request_model": {
                "kernel_frac": {k: round(req_model[k] / means[k], 4) for k in means},
                "step_frac": sum(req_model.values()) / (ms_per_step),
                "model_ms": {k: round(v, 4) for k, v in req_model.items()},
                "line_ps": a_ps, "sector_ps": b_ps, "probe_gbs": {"32": g32, "128": g128},
                "applies": tables_bytes <= L2_BYTES,
                "note": "t = E * sum over gathered rows (line_ps * 128 B lines + sector_ps * "
                        "32 B sectors), costs fitted live from the 32 B and 128 B L2 probe "
                        "points: the ceiling for request-bound gathers from L2-resident tables"},
            "step_roofline": {"algorithmic_bytes": step_bytes,
                              "achieved": step_bytes / (ms_per_step / 1e3) / 1e9,
                              "frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "GEdges/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "mode": ("pinned host buffers through the C-ABI; every step copies its own "
                             "inputs H2D and outputs D2H inside the timed region, double-buffered "
                             "so step i+1's upload and step i-1's download overlap step i's "
                             f"kernels; {h2d / 1e6:.0f} MB of fresh input per step")
                            if not sharded else
                            ("pinned host buffers through the C-ABI; each rank uploads its own "
                             "rows of the inputs and downloads its own rows of the outputs every "
                             "step, NCCL all-gathers inside the step; max over ranks"),
                    "serial_value": e2e_serial,
                    "graph_value": (e2e_graph or {}).get("value"),
                    "graph_mode": "the serial step (copies + 3 kernels) captured in one CUDA "
                                  "graph and replayed, L2 flushed between replays"
                                  + (f"; capture failed: {e2e_graph['error']}"
                                     if e2e_graph and "error" in e2e_graph else ""),
                    "serial_mode": "one step at a time (copies overlap only within the step), "
                                   "L2 flushed between steps"},
            "layer": layer_out,
            "fwd_strategy_ms": ablation,
            "bwd_strategy_ms": bwd_ablation,
            # fwd (or one per source block + the merge when phased), pass A, pass B
            "gpu_launches": ((world + 1) if phased else 1) * args.steps + 2 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(out))
    if sharded:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Worker for tests/test_shard_multiproc_gpu.py (launched by
torch.distributed.run, every rank on the one GPU, gloo process group).

The row-sharded layer step across real processes: each rank owns a block of
destination rows / source columns (shard.RowShard), holds ONLY its own block
of the source-side tables (the other blocks zeroed), obtains the rest through
the same all-gathers bench.py's sharded step uses (V and Q|el before the
forward; dO, K (dot) and the softmax records before pass B), runs the three
kernels on its rows / columns, and all-gathers its outputs.  Every rank then
checks O, dQ|del, dK|der and dV against the unsharded 1-GPU result BITWISE
(owner-computes keeps every per-row / per-column reduction order) and prints
SHARD-OK.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2411_16127_b200 import fused  # noqa: E402
from paper_2411_16127_b200.shard import RowShard, all_gather_rows  # noqa: E402


def graph(seed=0, n=3000):
    rng = np.random.default_rng(seed)
    deg = np.maximum(0, np.round(1500 * (np.arange(n) + 1.0) ** -0.6)).astype(np.int64)
    dst = np.repeat(rng.permutation(n), deg)
    src = rng.integers(0, n, dst.shape[0])
    key = np.unique(np.concatenate([dst * n + src, src * n + dst]))  # out-hubs too
    return oracle.from_coo(n, key % n, key // n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gat", choices=["gat", "gat_layer", "gt", "agnn"])
    ap.add_argument("--phased", action="store_true",
                    help="source-phased forward: per-block broadcasts, one forward per source "
                         "block, gf_attn_merge_parts (equal to 1 GPU up to the merge's rounding)")
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    H, D = (1, 128) if args.model == "agnn" else ((8, 16) if args.model == "gt" else (8, 8))
    variant = "add" if args.model.startswith("gat") else "dot"
    layer_form = args.model == "gat_layer"
    spec = fused.AttnSpec(variant, H, D, scale=0.25, slope=0.2, l2=args.model == "agnn",
                          logits_from_v=layer_form)
    g = graph()
    rng = np.random.default_rng(7)
    w = spec.qk_width
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=dev)  # noqa: E731
    if layer_form:
        Q, K = t(rng.uniform(-1, 1, (1, H * D))), t(rng.uniform(-1, 1, (1, H * D)))
    else:
        Q, K = t(rng.uniform(-1.5, 1.5, (g.n, w))), t(rng.uniform(-1.5, 1.5, (g.n, w)))
    V, dO = t(rng.uniform(-1, 1, (g.n, H * D))), t(rng.uniform(-1, 1, (g.n, H * D)))

    # the unsharded 1-GPU result
    full = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row,
                                           cta_threshold=64)
    O1, st1 = fused.attn_forward(full, spec, Q, K, V)
    dQ1, dK1, dV1 = fused.attn_backward(full, spec, Q, K, V, O1, st1, dO)

    # this rank's shard: only its own block of every node table is valid
    h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    sh = RowShard.build(g.n, h(g.row_ptr), h(g.col), h(g.csc_ptr), h(g.csc_row), rank, world)
    node_qk = not layer_form

    def own_only(x):
        p = sh.to_padded(x)
        keep = torch.zeros(p.shape[0], dtype=torch.bool, device=dev)
        keep[sh.block] = True
        p[~keep] = 0
        return p

    Vp, dOp = own_only(V), own_only(dO)
    Qp, Kp = (own_only(Q), own_only(K)) if node_qk else (Q, K)
    dg = sh.device_graph(cta_threshold=64)
    Op = torch.zeros_like(Vp)
    stp = torch.zeros(sh.n_padded, H, 4, device=dev)
    dQp = torch.zeros(sh.n_padded, w, device=dev)
    dKp = torch.zeros_like(dQp)
    dVp = torch.zeros_like(Vp)
    if args.phased:  # as bench.py's phased step: broadcasts per owner block, own block first
        from paper_2411_16127_b200 import shard as shard_mod

        parts = shard_mod.source_parts(sh, cta_threshold=64)
        O_parts, rec_parts = shard_mod.part_buffers(parts, spec, device=dev)
        R = sh.R
        blocks = {b: [dist.broadcast(t[b * R:(b + 1) * R], src=b, async_op=True)
                      for t in (Vp,) + ((Qp,) if node_qk else ())] for b in range(world)}
        for b in shard_mod.phase_order(sh):
            if b != rank:
                for wk in blocks[b]:
                    wk.wait()
            shard_mod.phase_forward(parts, b, spec, Qp, Kp, Vp, O_parts, rec_parts)
        for b in range(world):
            for wk in blocks[b]:
                wk.wait()
        shard_mod.merge_phases(parts, spec, O_parts, rec_parts, Op, stp)
    else:
        for x in (Vp,) + ((Qp,) if node_qk else ()):  # exchange 1: source rows for fwd / pass A
            all_gather_rows(x, sh)
        fused.attn_forward(dg, spec, Qp, Kp, Vp, O=Op, stats=stp)
    fused.attn_backward_rows(dg, spec, Qp, Kp, Vp, Op, stp, dOp, dKp)
    for x in (dOp, stp) + ((Kp,) if variant == "dot" else ()):  # exchange 2: pass B's gathers
        all_gather_rows(x, sh)
    fused.attn_backward_cols(dg, spec, Qp, Kp, Vp, stp, dOp, dQp, dVp)
    for x in (Op, dQp, dKp, dVp):  # outputs: every rank's owned rows
        all_gather_rows(x, sh)
    torch.cuda.synchronize()
    for a, b, name in ((O1, Op, "O"), (dQ1, dQp, "dQ"), (dK1, dKp, "dK"), (dV1, dVp, "dV")):
        b = sh.from_padded(b)
        if args.phased:  # merged partials: equal up to fp32 rounding of the merge
            err = float(((a - b).abs() / torch.clamp(torch.maximum(a.abs(), b.abs()), min=1)).max())
            if not err <= 2e-5:
                raise SystemExit(f"rank {rank}: {name} differs from 1 GPU (rel {err})")
        elif not torch.equal(a, b):
            err = float((a - b).abs().max())
            raise SystemExit(f"rank {rank}: {name} differs from 1 GPU (max abs {err})")
    print(f"SHARD-OK rank {rank}/{world} {args.model}{' phased' if args.phased else ''}",
          flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

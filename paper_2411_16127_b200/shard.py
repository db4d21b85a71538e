"""Row-sharded multi-GPU execution of the fused layer.

Partition: contiguous node ranges balanced by in+out edge count; rank k owns
nodes [b_k, b_{k+1}): the in-edges of its nodes (CSR rows: forward and
backward pass A) and the out-edges of its nodes (CSC columns: pass B),
owner-computes on both sides, no atomics, no reduce-scatter.

Id space: nodes are relabelled new(v) = k*R + (v - b_k) with R = max shard
size, so every rank's node slice is one contiguous block of a padded table of
world*R rows.  NCCL all-gathers of per-rank slices then land in place
(all_gather_into_tensor with the rank's block as input), and because the
relabelling is monotonic, every row keeps its in-edge order and every column
its out-edge order — results are bitwise those of one GPU.

Per layer step the exchanges are:
  forward : all-gather of the source-side projected rows (V | Q, el)
  backward: all-gather of dO and the softmax records of the destination rows
            (pass B needs them for every out-edge of the owned columns)
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


def partition(n: int, row_ptr: torch.Tensor, csc_ptr: torch.Tensor, world: int) -> list[int]:
    """Node boundaries b_0=0 <= ... <= b_world=n balancing in+out edges."""
    cum = (row_ptr.to(torch.int64) + csc_ptr.to(torch.int64)).cpu()
    total = int(cum[-1])
    bounds = [0]
    for k in range(1, world):
        target = total * k // world
        b = int(torch.searchsorted(cum, torch.tensor([target]), right=False)[0])
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return bounds


@dataclass
class RowShard:
    rank: int
    world: int
    n: int                 # original node count
    bounds: list           # node boundaries, len world+1
    R: int                 # padded rows per rank
    row_ptr: torch.Tensor  # int32 [world*R + 1]: CSR of the owned rows (padded ids)
    col: torch.Tensor      # int32 [e_csr]
    csc_ptr: torch.Tensor  # int32 [world*R + 1]: CSC of the owned columns
    csc_row: torch.Tensor  # int32 [e_csc]
    e_total: int = 0       # edges of the unsharded graph (sets the multi-CTA split_len)

    @property
    def n_padded(self) -> int:
        return self.world * self.R

    @property
    def lo(self) -> int:
        return self.bounds[self.rank]

    @property
    def hi(self) -> int:
        return self.bounds[self.rank + 1]

    @property
    def rows(self) -> slice:
        """This rank's block of a padded node table."""
        return slice(self.rank * self.R, self.rank * self.R + (self.hi - self.lo))

    @property
    def block(self) -> slice:
        return slice(self.rank * self.R, (self.rank + 1) * self.R)

    # ------------------------------------------------------------ building --
    @classmethod
    def build(cls, n, row_ptr, col, csc_ptr, csc_row, rank, world) -> "RowShard":
        """From the full canonical CSR/CSC (int64/int32 tensors on any device)."""
        bounds = partition(n, row_ptr, csc_ptr, world)
        R = max(1, max(bounds[k + 1] - bounds[k] for k in range(world)))
        dev = col.device
        b = torch.tensor(bounds, dtype=torch.int64, device=dev)

        def relabel(ids):
            ids = ids.to(torch.int64)
            k = torch.searchsorted(b, ids, right=True) - 1
            return (k * R + (ids - b[k])).to(torch.int32)

        def side(ptr, idx):
            lo, hi = bounds[rank], bounds[rank + 1]
            p = ptr.to(torch.int64)
            e0, e1 = int(p[lo]), int(p[hi])
            out = torch.full((world * R + 1,), e1 - e0, dtype=torch.int64, device=dev)
            out[: rank * R + 1] = 0
            out[rank * R: rank * R + (hi - lo) + 1] = p[lo: hi + 1] - e0
            return out.to(torch.int32), relabel(idx[e0:e1])

        rp, c = side(row_ptr, col)
        cp, cr = side(csc_ptr, csc_row)
        return cls(rank, world, n, bounds, R, rp, c, cp, cr, int(row_ptr[-1]))

    def to_padded(self, x: torch.Tensor) -> torch.Tensor:
        """Full node table (original ids) -> padded table (world*R rows)."""
        out = torch.zeros((self.n_padded,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        for k in range(self.world):
            lo, hi = self.bounds[k], self.bounds[k + 1]
            out[k * self.R: k * self.R + hi - lo] = x[lo:hi]
        return out

    def from_padded(self, xp: torch.Tensor) -> torch.Tensor:
        parts = [xp[k * self.R: k * self.R + self.bounds[k + 1] - self.bounds[k]]
                 for k in range(self.world)]
        return torch.cat(parts, 0)

    def device_graph(self, cta_threshold: int = 0, stream=None):
        """gf_graph_t over the padded id space; empty (foreign) rows skipped.
        Super rows are split over CTAs exactly as in the unsharded graph
        (split_len from the total edge count), so owned rows / columns keep
        the 1-GPU reduction order."""
        from .fused import DeviceGraph, default_split_len

        dg = DeviceGraph.from_split(self.n_padded, self.row_ptr, self.col, self.csc_ptr,
                                    self.csc_row, cta_threshold=cta_threshold, skip_empty=True,
                                    stream=stream)
        if self.e_total:
            dg.set_split_len(default_split_len(self.e_total, cta_threshold), stream=stream)
        return dg


def all_gather_rows(table: torch.Tensor, shard: RowShard, group=None, async_op=False):
    """In-place all-gather of every rank's block of a padded node table."""
    import torch.distributed as dist

    blk = table[shard.block]
    return dist.all_gather_into_tensor(table, blk, group=group, async_op=async_op)


def block_views(tables: list, shard: RowShard) -> list:
    """Destinations of this rank's block for a producer that writes every
    rank's copy of a padded table: [own table's block, then the same rows of
    each peer's table in rank order].  `tables[k]` is rank k's table (a
    peer-mapped view for k != rank)."""
    if len(tables) != shard.world:
        raise ValueError("block_views: one table per rank expected")
    order = [shard.rank] + [k for k in range(shard.world) if k != shard.rank]
    return [tables[k][shard.block] for k in order]


class PeerTables:
    """Padded node tables in symmetric memory (torch.distributed.
    _symmetric_memory): every rank's copy is addressable from every GPU
    through NVLink / NVSwitch peer mappings, so the kernel that produces a
    rank's block writes it straight into all copies (gf_gemm_bcast: the
    projection with its all-gather fused into the epilogue) and a device-side
    barrier replaces the collective.  One symmetric buffer holds all tables."""

    def __init__(self, shard: RowShard, widths: dict, dtype=torch.float32, device=None,
                 group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.shard = shard
        group = group if group is not None else dist.group.WORLD
        n = shard.n_padded
        total = n * sum(widths.values())
        self.buf = symm_mem.empty(total, dtype=dtype, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, group)
        # the tensor's place inside the symmetric allocation (same on every rank)
        self.storage_offset = int(getattr(self.hdl, "offset", 0)) // self.buf.element_size()
        self.peer_bufs = [self.buf if k == shard.rank else
                          self.hdl.get_buffer(k, (total,), dtype, self.storage_offset)
                          for k in range(shard.world)]
        self.offsets = {}
        off = 0
        for name, w in widths.items():
            self.offsets[name] = (off, w)
            off += n * w

    def _table(self, buf, name):
        off, w = self.offsets[name]
        return buf[off: off + self.shard.n_padded * w].view(self.shard.n_padded, w)

    def table(self, name) -> torch.Tensor:
        """This rank's full padded table."""
        return self._table(self.buf, name)

    def dests(self, name) -> list:
        """gemm_bcast destinations of this rank's block (own first)."""
        return block_views([self._table(b, name) for b in self.peer_bufs], self.shard)

    def selftest(self):
        """End-to-end check of the peer addressing: every rank writes rank+1
        into its block of every copy of the first table, barrier, and every
        block of the local copy must then hold its owner's value.  Raises on a
        mismatch (the caller falls back to the NCCL exchange)."""
        import torch.distributed as dist

        name = next(iter(self.offsets))
        R = self.shard.R
        t = self.table(name)
        self.barrier()
        for d in self.dests(name):
            d.fill_(float(self.shard.rank + 1))
        self.barrier()
        got = t.view(self.shard.world, R, -1)[:, :, 0].cpu()
        want = torch.arange(1, self.shard.world + 1, dtype=got.dtype)[:, None].expand_as(got)
        ok = torch.equal(got, want)
        self.barrier()  # every rank passes every barrier whatever its verdict
        # all ranks take the same decision (a rank falling back alone would
        # leave the others waiting in a device barrier)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=t.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            raise RuntimeError("PeerTables.selftest: peer writes did not land in every copy")

    def barrier(self):
        """Device-side barrier on the current stream: every rank's writes
        issued before it are visible to every rank after it."""
        self.hdl.barrier(channel=0)


# ------------------------------------------------- source-phased forward --
# The forward gathers source rows of every rank, so its all-gather cannot
# simply run under it.  But CSR rows are sorted by source and every rank's
# sources are one contiguous id block, so each row's in-edges split into P
# contiguous slices by source block.  Running the forward once per block — the
# local block first, then each block as its rows arrive — and merging the
# normalised partials (gf_attn_merge_parts) overlaps the exchange with the
# forward ("chunked all-gather overlapped with compute on locally-sourced
# edges first").  Deterministic; equal to the one-pass forward
# up to the merge's rounding (the one-pass path stays bitwise equal to 1 GPU).

@dataclass
class SourceParts:
    shard: RowShard
    graphs: list    # DeviceGraph of the rank's rows restricted to source block k
    row_ptrs: list  # int32 [n_padded + 1] row pointer of each part (device)


def source_split(shard: RowShard) -> list:
    """[(row_ptr_k, col_k)] per source block k: the rank's CSR restricted to
    in-edges whose (padded) source id lies in [k R, (k+1) R), rows and each
    row's sources in their original order (int32, on the shard's device)."""
    R, P, n = shard.R, shard.world, shard.n_padded
    rp = shard.row_ptr.to(torch.int64)
    col = shard.col.to(torch.int64)
    dev = col.device
    deg = rp[1:] - rp[:-1]
    row_of = torch.repeat_interleave(torch.arange(n, device=dev), deg)
    blk = col // R
    counts = torch.zeros(n * P, dtype=torch.int64, device=dev)
    counts.index_add_(0, row_of * P + blk, torch.ones_like(blk))
    counts = counts.view(n, P)
    out = []
    for k in range(P):
        ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        ptr[1:] = torch.cumsum(counts[:, k], 0)
        out.append((ptr.to(torch.int32), col[blk == k].to(torch.int32)))
    return out


def source_parts(shard: RowShard, cta_threshold: int = 0, stream=None) -> SourceParts:
    from .fused import DeviceGraph

    n = shard.n_padded
    dev = shard.col.device
    empty_ptr = torch.zeros(n + 1, dtype=torch.int32, device=dev)
    dummy = torch.zeros(1, dtype=torch.int32, device=dev)
    graphs, ptrs = [], []
    for ptr, ck in source_split(shard):
        ptrs.append(ptr)
        graphs.append(DeviceGraph.from_split(n, ptr, ck if ck.numel() else dummy, empty_ptr,
                                             dummy, cta_threshold=cta_threshold, skip_empty=True,
                                             stream=stream))
    return SourceParts(shard, graphs, ptrs)


def part_buffers(parts: SourceParts, spec, dtype=torch.float32, device=None):
    """Row-block-sized partial outputs: one R x F O and R x H x 4 record table
    per part (the kernels address them in the padded id space through a base
    pointer offset by the rank's first row)."""
    R = parts.shard.R
    O = [torch.empty(R, spec.F, dtype=dtype, device=device) for _ in parts.graphs]
    rec = [torch.empty(R, spec.heads, 4, dtype=dtype, device=device) for _ in parts.graphs]
    return O, rec


def phase_forward(parts: SourceParts, k: int, spec, Q, K, V, O_parts, rec_parts, stream=None):
    """Forward over source block k's in-edges of the rank's rows into part k."""
    import ctypes as C

    from ._capi import check, lib
    from .fused import _stream

    sh = parts.shard
    es = V.element_size()
    row0 = sh.rank * sh.R
    o_base = O_parts[k].data_ptr() - row0 * spec.F * es
    r_base = rec_parts[k].data_ptr() - row0 * spec.heads * 4 * es
    d = spec.desc(V.dtype)
    check(lib().gf_attn_fwd(parts.graphs[k].handle, C.byref(d), C.c_void_p(Q.data_ptr()),
                            C.c_void_p(K.data_ptr()), C.c_void_p(V.data_ptr()),
                            C.c_void_p(o_base), C.c_void_p(r_base), None, _stream(stream)),
          "gf_attn_fwd (phase)")


def merge_phases(parts: SourceParts, spec, O_parts, rec_parts, O, stats, stream=None):
    """O / records of the rank's block from the per-block partials."""
    from .fused import attn_merge_parts

    sh = parts.shard
    blk = sh.block
    ptrs = [p[blk.start: blk.stop + 1] for p in parts.row_ptrs]
    attn_merge_parts(spec, ptrs, O_parts, rec_parts, O[blk], stats[blk], stream=stream)


def phase_order(shard: RowShard) -> list:
    """Own block first (its rows are local), then the others in rank order."""
    return [shard.rank] + [k for k in range(shard.world) if k != shard.rank]

// Internal shared definitions for libgraphfuse_cuda (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "gf_cuda.h"
#include "gf_policy.h"

namespace gfb {

// Kernel variant of the GAT layer (gf_attn_desc flag GF_FLAG_LOGITS_FROM_V):
// additive scores whose logits are linear in the gathered V row itself,
// el[u,h] = <V[u,h,:], a_l[h,:]>, er[v,h] = <V[v,h,:], a_r[h,:]> (models.hpp:
// 116-125, V = H), so no el table is gathered per edge.  Q / K carry a_l / a_r
// (H x D, the layout of a V row).  Internal: not a gf_attn_desc.variant value.
constexpr int GF_ADDV = 2;
// The same layer form tuned for gathered tables far beyond L2 (HBM-bound, short
// rows: C5): more resident warps, fewer edges in flight per warp
// (GF_MINB_FWD_H / GF_U_FWD_H); selected by the forward launcher per graph.
constexpr int GF_ADDV_HBM = 3;
__host__ __device__ constexpr bool is_addv(int v) { return v == GF_ADDV || v == GF_ADDV_HBM; }

// ------------------------------------------------------------------ errors --
void set_error(const std::string& msg);

#define GF_CHECK_CUDA(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::gfb::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));          \
      return GF_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define GF_CHECK_LAUNCH(what)                                                        \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::gfb::set_error(std::string("launch ") + (what) + ": " + cudaGetErrorString(_e)); \
      return GF_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

// ----------------------------------------------------------------- scratch --
// Stream-ordered scratch (cudaMallocFromPoolAsync) from a library-private
// memory pool per device whose release threshold (8 GiB) keeps freed scratch
// mapped across synchronisations: with a threshold of 0 every sync hands it
// back to the driver and the next call pays for a fresh physical mapping
// (measured: +5.6 ms per unfused AGNN backward on C3).  The device's default
// pool (the host application's) is untouched; gf_scratch_trim() releases.
cudaError_t scratch_alloc_raw(void** p, size_t bytes, cudaStream_t s);
template <class P>
inline cudaError_t scratch_alloc(P** p, size_t bytes, cudaStream_t s) {
  return scratch_alloc_raw(reinterpret_cast<void**>(p), bytes, s);
}

// ------------------------------------------------------------------- graph --
// Device-resident topology: int32 CSR (dst rows -> src) and CSC (src cols ->
// dst), plus the bi-level schedules (degree-descending orders with bucket
// counts) for the row pass (forward, backward pass A) and the column pass
// (backward pass B).
struct DevGraph {
  int32_t n = 0, e = 0;
  int32_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  int32_t* csc_ptr = nullptr;
  int32_t* csc_row = nullptr;
  int32_t* row_order = nullptr;
  int32_t* col_order = nullptr;
  // per schedule slot {node, first edge, end edge, 0}: one 16 B load replaces
  // the dependent order -> pointer loads of a row's prologue
  int4* row_sched = nullptr;
  int4* col_sched = nullptr;
  int32_t cta_threshold = 0;
  int32_t n_cta_rows = 0, n_empty_rows = 0;
  int32_t n_cta_cols = 0, n_empty_cols = 0;
  // rows / columns with 1 <= degree <= kSmallDegree: they sit just before the
  // empty ones in the order and are packed several per warp (one lane group
  // each) by the fast kernels
  int32_t n_small_rows = 0, n_small_cols = 0;
  int64_t max_in = 0, max_out = 0;
  int device = 0;
  int32_t* coo_dst = nullptr;   // CSR-order destination per edge (built on first use by
                                // the edge-parallel strategies; graph-owned)
  int32_t* csc_perm = nullptr;  // CSC slot -> CSR edge id (reference csc_edge_perm), built
                                // on first use by the unfused backward ops; graph-owned
  // Multi-CTA split of super rows / columns: the CTA bucket's blocks, one
  // int4 {slot, slice, slices, first partial} per block.  A row of degree d
  // takes ceil(d / split_len) CTAs (split_len = max(cta_threshold,
  // E / (148 * 4))); split rows publish per-slice partial states that the
  // last-arriving CTA merges in slice order (gf_attn_fwd.cuh split_publish).
  int4* row_cta = nullptr;
  int4* col_cta = nullptr;
  int32_t row_cta_blocks = 0, col_cta_blocks = 0;  // CTA-bucket blocks
  int32_t row_parts = 0, col_parts = 0;            // partial slots of split rows / columns
  int32_t e_csc = 0;        // CSC edge count (== e unless row-sharded)
  bool skip_empty = false;  // do not visit rows / columns without edges
  /// Rows (resp. columns) a pass visits: the empty ones trail the order.
  int32_t active_rows() const { return skip_empty ? n - n_empty_rows : n; }
  int32_t active_cols() const { return skip_empty ? n - n_empty_cols : n; }
};

// Occupancy vs memory-level parallelism of the latency-bound gathers, per
// kernel: MINB = minimum resident 256-thread CTAs per SM requested from ptxas
// (register cap 65536 / (256 * MINB)), U = edges in flight per lane.  Tuned
// on B200 with scripts/ab_variants.sh (profiles/README.md): one-chunk lanes
// (GAT 8x8) fwd/pass A MINB 3, U 4; pass B MINB 4, U 2; two-chunk lanes
// (GT 8x16) MINB 2, U 1 for all three.
#ifndef GF_MINB_FWD
#define GF_MINB_FWD 3
#endif
#ifndef GF_U_FWD
#define GF_U_FWD 4
#endif
#ifndef GF_MINB_ROWS
#define GF_MINB_ROWS 3
#endif
#ifndef GF_U_ROWS
#define GF_U_ROWS 4
#endif
#ifndef GF_MINB_COLS
#define GF_MINB_COLS 4
#endif
#ifndef GF_U_COLS
#define GF_U_COLS 2
#endif
// A/B switches for the forward's row prologue (profiles/README.md).
// First row's {node, begin, end}: 1 = one 16 B schedule-entry load, 0 = the
// order -> pointer loads.  A/B on B200 (profiles/README.md): the forward is
// faster with 0 (C4 2.40 -> 2.16 ms), pass A with 1 (C4 2.22 -> 2.15 ms).
#ifndef GF_SCHED16_FWD
#define GF_SCHED16_FWD 0
#endif
#ifndef GF_SCHED16_ROWS
#define GF_SCHED16_ROWS 1
#endif
#ifndef GF_ROWPIPE
#define GF_ROWPIPE 1  // software-pipelined warp rows (rows_per_warp)
#endif
#ifndef GF_MINB2
#define GF_MINB2 2
#endif
#ifndef GF_U2
#define GF_U2 1
#endif
#ifndef GF_MINB_FWD_V
#define GF_MINB_FWD_V GF_MINB_FWD  // GAT layer form (GF_ADDV) forward
#endif
#ifndef GF_MINB_ROWS_V
#define GF_MINB_ROWS_V 4  // GAT layer form pass A (C4 1.91 -> 1.83 ms, C5 GAT 3.43 -> 3.06)
#endif
#ifndef GF_MINB_FWD_H
#define GF_MINB_FWD_H 4
#endif
#ifndef GF_U_FWD_H
#define GF_U_FWD_H 2
#endif
#ifndef GF_U_FWD_V
#define GF_U_FWD_V GF_U_FWD  // GAT layer form (GF_ADDV) forward
#endif
#ifndef GF_U_DOT1
#define GF_U_DOT1 2  // dot scores with one-chunk lanes (e.g. GT 8x8): Q and V rows per slot
#endif

#ifndef GF_U_DOT1_COLS
#define GF_U_DOT1_COLS 1  // ... pass B: one slot (dO + K rows) in flight, no spills
#endif

#ifndef GF_MINB_DOT1_COLS
#define GF_MINB_DOT1_COLS 3  // pass B, dot scores, one-chunk lanes: dV + dQ accumulators
#endif

#ifndef GF_U_ROWS_V
#define GF_U_ROWS_V 2  // GAT layer form pass A
#endif
#ifndef GF_U2_PK
#define GF_U2_PK 1  // packed rows of two-chunk lanes (A/B knob)
#endif

constexpr int kDefaultCtaThreshold = 1024;  // floor of the automatic threshold
// Automatic CTA-row threshold: a row gets a whole CTA once it holds more than
// ~1/8 of the edges one resident warp processes over the kernel (E / (148 SMs
// x 24 warps)), so no single warp row outlasts the launch, while rows below
// that keep the cheaper warp path (C4 sweep, profiles/ab_r1_cta_threshold.txt:
// 1024 -> 17.1, 3072-16384 -> 17.4-17.7 GEdges/s).  Clamped to [1024, 16384].
inline int auto_cta_threshold(int64_t e) {
  const int64_t t = e / (148 * 24 * 8);
  return static_cast<int>(t < kDefaultCtaThreshold ? kDefaultCtaThreshold : (t > 16384 ? 16384 : t));
}
constexpr int kSmallDegree = 8;  // packed (sub-warp) bucket: degree 1..8

// Warp-bucket rows per warp: software-pipelined row prologues pay off for
// short rows (average degree <= 64) but only while every SM still gets ~4
// waves of resident warps (148 SMs x 24 warps); otherwise one row per warp.
inline int rows_per_warp(int64_t edges, int64_t nodes, int64_t warp_rows) {
  if (edges > 64 * std::max<int64_t>(1, nodes)) return 1;
  const int64_t r = warp_rows / (148 * 24 * 4);
  return r >= 8 ? 8 : r >= 4 ? 4 : r >= 2 ? 2 : 1;
}
constexpr int kWarpsPerBlock = 8;  // 256-thread CTAs for every attention kernel

// Programmatic dependent launch (PDL) for the attention kernels: launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel's CTAs may be
// scheduled while the previous kernel in the stream is still finishing; every
// fast kernel executes griddepcontrol.wait (pdl_wait) before its first global
// memory access, so it still observes all of the previous kernel's writes,
// and pdl_launch lets the next kernel be scheduled early.  Hides the launch
// latency between fwd -> pass A -> pass B (small graphs).  GF_PDL=0 disables.
bool pdl_enabled();
template <typename Kern, typename Arg>
cudaError_t launch_k(Kern k, int blocks, int threads, cudaStream_t s, const Arg& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, a);
}
// Small graphs (E below this) prefetch their gathered node tables into L2 at
// kernel entry: with L2 cold the passes are bound by dependent DRAM round
// trips, and L2 hits cut each gather's latency (GF_L2_PREFETCH=0 disables).
constexpr int64_t kPrefetchMaxEdges = int64_t(4) << 20;
constexpr int64_t kPrefetchMaxBytes = int64_t(96) << 20;
bool l2_prefetch_enabled();

// Edges per CTA slice of a split row: no CTA of a pass holds more than ~1/4
// of one SM's share of the edges (148 SMs), and never fewer than a CTA row.
// GF_SPLIT_LEN=<edges> overrides (A/B; a huge value disables splitting).
inline int64_t split_len(int64_t e, int cta_threshold) {
  const char* env = std::getenv("GF_SPLIT_LEN");
  if (env && *env) return std::max<int64_t>(1, std::atoll(env));
  return std::max<int64_t>(std::max(cta_threshold, 1), (e + 148 * 4 - 1) / (148 * 4));
}

// ---------------------------------------------------------- kernel params --
// Lane geometry of the fast path (see fast_shape): a lane owns CPL chunks of
// CB bytes of ONE head; LPH lanes share a head; LPE = H * LPH lanes per edge.
template <typename T>
struct FwdArgs {
  const int32_t* ptr;    // CSR row pointer
  const int32_t* idx;    // CSR column (source) ids
  const int32_t* order;  // row schedule
  int n, n_cta;
  int H, D, F, LPH;
  int l2;
  T scale, slope;
  const int4* sched = nullptr;  // {node, begin, end} per slot (fast kernels)
  const T* Q;  // dot: N x F; add: el N x H
  const T* K;  // dot: N x F; add: er N x H
  const T* V;
  T* O;
  T* stats;  // N x H x 4 records (gf_device.cuh Rec)
  int pk0 = 0, wblocks = 0;  // packed bucket: first slot; #blocks of the warp bucket
  int rpw = 1;               // warp-bucket rows per warp (software-pipelined prologues)
  int n_small = 0, n_empty = 0;  // bucket counts of the order being walked (rows or columns)
  int64_t e = 0;                 // edges of that view (rows_per_warp)
  const T* ES = nullptr;  // E x H edge scores (PMF) / probabilities (unfused), CSR order
  const int32_t* eperm = nullptr;  // MODE 3: slot -> CSR edge id of ES (CSC passes)
  // multi-CTA split rows (DevGraph::row_cta); cta_tab == nullptr: one CTA per
  // CTA-bucket row (block b -> slot b)
  const int4* cta_tab = nullptr;
  int cta_blocks = 0, parts = 0;
  T* part = nullptr;           // parts x LPE x (2 + NE) slice states
  unsigned* part_cnt = nullptr;  // arrivals per split row (indexed by its first partial)
  // small graphs: node tables the launch gathers, prefetched into L2 by every
  // thread's first instructions (see l2_prefetch_tables)
  const void* pf_ptr[3] = {nullptr, nullptr, nullptr};
  int64_t pf_len[3] = {0, 0, 0};
  uint64_t pol = kPolicyEvictLast;  // L2 policy word of the gathers (gf_policy.h)
};

template <typename T>
struct BwdArgs {
  const int32_t* ptr;
  const int32_t* idx;
  const int32_t* order;
  int n, n_cta;
  int H, D, F, LPH;
  int l2;
  T scale, slope;
  const int4* sched = nullptr;
  const T* Q;
  const T* K;
  const T* V;
  const T* O;
  const T* dO;
  T* stats;  // records; pass A writes delta, pass B reads them
  T* dQ;     // pass B (dot) / del (add)
  T* dK;     // pass A (dot) / der (add)
  T* dV;     // pass B
  int pk0 = 0, wblocks = 0;  // packed bucket: first slot; #blocks of the warp bucket
  int rpw = 1;               // warp-bucket rows per warp
  const int4* cta_tab = nullptr;  // multi-CTA split (as FwdArgs)
  int cta_blocks = 0, parts = 0;
  T* part = nullptr;
  unsigned* part_cnt = nullptr;
  const void* pf_ptr[3] = {nullptr, nullptr, nullptr};  // L2 prefetch (as FwdArgs)
  int64_t pf_len[3] = {0, 0, 0};
  uint64_t pol = kPolicyEvictLast;  // as FwdArgs
};

// Launchers (defined in gf_attn_fwd.cuh / gf_attn_bwd.cuh).
template <typename T>
int launch_fwd(const DevGraph& g, const FwdArgs<T>& a, int variant, cudaStream_t s);
template <typename T>
int launch_materialize_p(const DevGraph& g, const FwdArgs<T>& a, int variant, T* P,
                         cudaStream_t s);
// Forward kernel modes: 0 = SMMF (compute scores), 1 = scores read from ES
// (PMF's fused softmax + SpMM), 2 = edge weights read from ES (plain SpMM:
// no softmax, O = scale * sum w V, no records), 3 = as 2 with the weight of
// slot i at ES[eperm[i]] (SpMM over the CSC view with CSR-ordered weights).
template <typename T>
int launch_fwd_mode(const DevGraph& g, const FwdArgs<T>& a, int variant, int mode, cudaStream_t s);
// Lazily built per-graph edge maps (gf_attn_strategies.cu / gf_unfused_ops.cu).
int ensure_coo_dst(DevGraph& g, cudaStream_t s);
int ensure_csc_perm(DevGraph& g, cudaStream_t s);
// Edge-parallel SDDMM into S[E x H] and the row softmax S -> P (+ records when
// a.stats != nullptr).
template <typename T>
int launch_sddmm_edges(DevGraph& g, const FwdArgs<T>& a, int variant, T* S, cudaStream_t s);
template <typename T>
int launch_softmax_rows(const DevGraph& g, const FwdArgs<T>& a, int variant, const T* S, T* P,
                        cudaStream_t s);
// Fusion strategies (gf_attn_strategies.cu).  ws: E*H (PMF) or 2*E*H
// (unfused without caller P) elements of scratch.
size_t strategy_workspace_bytes(const DevGraph& g, int heads, int elem, int strategy, bool have_p);
template <typename T>
int launch_fwd_strategy(DevGraph& g, const FwdArgs<T>& a, int variant, int strategy, T* P, T* ws,
                        cudaStream_t s);
// passes: bit 0 = pass A (CSR rows), bit 1 = pass B (CSC columns).
template <typename T>
int launch_bwd(const DevGraph& g, BwdArgs<T> a, int variant, int passes, cudaStream_t s);

// Fast-path geometry.  Chunk bytes CB: 32 when a head row is a multiple of
// 32 B (256-bit loads), else 16.  Chunks per head CPH = D*sizeof(T)/CB; a lane
// owns CPL = min(CPH, 2) chunks and LPH = CPH / CPL lanes share a head, so
// lanes per edge LPE = H * LPH (a power of two <= 32).
struct FastShape {
  bool ok = false;
  int cb = 0, lpe = 0, cpl = 0, lph = 0;
};
// Heads of >= 2 chunks take two chunks per lane.  One chunk per lane (twice
// the lanes per edge, fewer registers) measured slower on every config, small
// graphs included (C2 0.71 -> 0.45, C3 0.94 -> 0.67, C5 GT 1.78 -> 1.17
// GEdges/s, profiles/r2/ab_r2_one_chunk_lanes.txt); GF_CPL=1 forces it (A/B).
FastShape fast_shape(int H, int D, int elem_bytes, int64_t edges);

}  // namespace gfb

// The opaque C handle is the device graph itself.
struct gf_graph_s : gfb::DevGraph {};

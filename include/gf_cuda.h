/* gf_cuda.h — C-ABI of the B200-native fused AT-GNN path (libgraphfuse_cuda.so).
 *
 * This is the drop-in boundary underneath the reference's C++ operator API
 * (namespace graphfuse, proj/include/graphfuse/ headers) and its
 * pybind11 module graphfuse._core (/root/reference/proj/bindings/module.cpp).
 * Plain pointers, sizes and an opaque graph handle; no torch or C++ types.
 * Every compute entry point takes DEVICE pointers and a cudaStream_t passed as
 * void*; nothing synchronises the stream except where stated.
 *
 * Conventions (identical to the reference):
 *   - edge u -> v; CSR rows are destinations listing in-neighbours sorted by
 *     source (graph.hpp:18-23); CSC columns are sources listing destinations
 *     sorted ascending (graph.cpp:43-55).
 *   - dot scores s = scale * <Q[u], K[v]> (query at the SOURCE, key at the
 *     destination, kernels.hpp:17-33); AGNN additionally L2-normalises Q and K
 *     rows per head with max(||x||, 1e-12) (kernels.hpp:50-61).
 *   - add (GAT) scores s = LeakyReLU(el[u] + er[v]) with x>=0 ? x : slope*x
 *     (kernels.hpp:36-47); backward derivative pre>0 ? 1 : slope
 *     (autograd.hpp:113).
 *   - per-destination softmax; empty rows give zero output (kernels.hpp:65-102).
 * Multi-head layout (the reference is single-head and is applied per head):
 *   dot: Q, K, dQ, dK are N x (H*D); add: el, er, del, der are N x H;
 *   V, O, dO, dV are N x (H*D); all row-major, element type `dtype`.
 *   stats is N x H x 4 softmax records {m, log2 l, aux, delta} per (row,
 *   head): m = a reference score at most 8 below the row max (the forward
 *   rescales its running sum lazily), l = sum exp(s - m) (so p is recomputed
 *   as exp((s - m) - log l) with full relative precision for any |s|; only
 *   the pair is meaningful, m + ln(2) log2 l = the row's log-sum-exp),
 *   aux = er (GAT) or 1/max(||K||, eps) (AGNN), delta = <dO, O> (written by
 *   backward pass A).  Base pointers must be 32-byte aligned for the 256-bit
 *   gather path (torch / cudaMalloc allocations are); other alignments fall
 *   back to the generic kernels.
 *
 * Errors: every function returns GF_OK (0) or a GF_ERR_* code; the message is
 * available from gf_last_error() (thread-local).  Launch failures are
 * reported, never swallowed; there is no CPU fallback.
 */
#ifndef GF_CUDA_H
#define GF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_OK 0
#define GF_ERR_INVALID 1  /* bad argument / shape (reference: KernelError, std::invalid_argument) */
#define GF_ERR_CUDA 2     /* CUDA runtime / launch failure */
#define GF_ERR_GRAPH 3    /* topology error (reference: GraphError) */
#define GF_ERR_UNSUPPORTED 4

#define GF_F32 0
#define GF_F64 1
#define GF_DOT 0 /* SddmmVariant::Dot (GT, AGNN) */
#define GF_ADD 1 /* SddmmVariant::Add (GAT) */

/* gf_attn_desc.reserved flags.
 * GF_FLAG_LOGITS_FROM_V (GF_ADD only): the GAT layer's attention logits are
 * linear in the projected features V = H (models.hpp:116-125): Q and K carry
 * a_l and a_r (H x D, the layout of one V row, 32-byte aligned) and the
 * kernels compute el[u,h] = <V[u,h,:], a_l[h,:]> from the V row they gather
 * anyway and er[v,h] = <V[v,h,:], a_r[h,:]> from the destination's own row,
 * instead of gathering an el table per edge.  Backward outputs are unchanged
 * (dQ|del, dK|der are N x H).  Paths other than the fused fast kernels
 * (strategies, P materialisation, generic shapes) compute el / er tables
 * once (gf_gat_logits) and run the table form. */
#define GF_FLAG_LOGITS_FROM_V 1

/* Fusion strategies (reference Strategy enum, schedule.hpp:12-18). */
#define GF_STRAT_SMMF 0     /* 1 launch, fused, nothing E x H in HBM (default)      */
#define GF_STRAT_PMF 1      /* edge-parallel SDDMM -> S[E x H]; fused softmax+SpMM  */
#define GF_STRAT_UNFUSED 2  /* SDDMM -> S; softmax -> P[E x H]; SpMM: 3 launches    */
#define GF_STRAT_BASELINE 3 /* feature-parallel fused kernel, rows in id order      */

typedef struct gf_graph_s* gf_graph_t;

/* Attention operator descriptor: SddmmKind (dense.hpp:48-62) + head shape. */
typedef struct gf_attn_desc {
  int32_t dtype;    /* GF_F32 | GF_F64 */
  int32_t variant;  /* GF_DOT | GF_ADD */
  int32_t l2;       /* AGNN: L2-normalise Q and K rows per head (dot only) */
  int32_t heads;    /* H >= 1 */
  int32_t head_dim; /* D >= 1 */
  int32_t reserved; /* flags (GF_FLAG_*); 0 = the reference's SddmmKind semantics */
  double scale;     /* dot only */
  double slope;     /* add only (LeakyReLU negative slope) */
} gf_attn_desc;

/* Degree-bucket schedule summary of a device graph (the bi-level scheduler). */
typedef struct gf_graph_info {
  int64_t num_nodes, num_edges;
  int64_t max_in_degree, max_out_degree;
  int32_t cta_threshold;   /* rows with degree >= this get a whole CTA (edge-split) */
  int32_t n_cta_rows;      /* CSR rows in the CTA bucket (lead the row order) */
  int32_t n_empty_rows;    /* CSR rows of degree 0 (trail the row order) */
  int32_t n_cta_cols;      /* CSC columns in the CTA bucket */
  int32_t n_empty_cols;
  int32_t device;
  int32_t n_small_rows;    /* CSR rows of degree 1..8: packed several per warp, one lane group
                              each (just before the empty rows in the order) */
  int32_t n_small_cols;
  int32_t cta_blocks_rows; /* CTA-bucket blocks of the row pass: > n_cta_rows when super rows
                              are split over several CTAs (multi-CTA split) */
  int32_t cta_blocks_cols;
} gf_graph_info;

const char* gf_last_error(void);
/* 1 if the library was built for (and can launch on) the current device. */
int gf_device_ok(void);

/* Memory plumbing for hosts that do not link the CUDA runtime themselves
 * (the C++ host layer and the pybind module use only this C-ABI).
 * gf_malloc / gf_free are stream-ordered on the legacy default stream (the
 * library's private pool): use the buffer on that stream or on a blocking
 * stream.  kind: 0 host->device, 1 device->host, 2 device->device.
 * gf_memcpy of >= 64 MiB between pageable host memory and the device goes
 * through a pinned staging ring (DMA of one chunk overlapping the host copy
 * of the previous one) and returns when the copy is complete. */
int gf_malloc(size_t bytes, void** out);
int gf_free(void* p);
int gf_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream);
int gf_memset(void* dst, int32_t value, size_t bytes, void* stream);
int gf_stream_sync(void* stream);

/* ---- topology (replaces the device half of graph.hpp:24-38 / graph.cpp:25-78) ----
 * From the reference's canonical host arrays (int64, as in graphfuse::Graph);
 * the CSC edge permutation is not needed on the device (the backward
 * recomputes attention instead of indexing a stored P).  cta_threshold <= 0
 * selects the automatic threshold clamp(E / 28416, 1024, 16384) (a row gets
 * a whole CTA once it holds ~1/8 of one resident warp's share of the edges).
 * Synchronises `stream` once (schedule build). */
int gf_graph_create(int64_t num_nodes, int64_t num_edges, const int64_t* csr_row_ptr,
                    const int64_t* csr_col_idx, const int64_t* csc_col_ptr,
                    const int64_t* csc_row_idx, int32_t cta_threshold, void* stream,
                    gf_graph_t* out);
/* Same from device int32 arrays (copied; caller keeps ownership of inputs). */
int gf_graph_create_device(int64_t num_nodes, int64_t num_edges, const int32_t* d_row_ptr,
                           const int32_t* d_col_idx, const int32_t* d_csc_ptr,
                           const int32_t* d_csc_row, int32_t cta_threshold, void* stream,
                           gf_graph_t* out);
/* Row-sharded graph (multi-GPU, §8(e)): the CSR (rows this rank owns, e_csr
 * edges) and the CSC (columns this rank owns, e_csc edges) may hold different
 * edge sets of the same node-id space.  flags & GF_GRAPH_SKIP_EMPTY: rows /
 * columns without edges are not visited at all (their outputs are left
 * untouched) — used when most rows belong to other ranks. */
#define GF_GRAPH_SKIP_EMPTY 1
int gf_graph_create_split(int64_t num_nodes, int64_t e_csr, const int32_t* d_row_ptr,
                          const int32_t* d_col_idx, int64_t e_csc, const int32_t* d_csc_ptr,
                          const int32_t* d_csc_row, int32_t cta_threshold, int32_t flags,
                          void* stream, gf_graph_t* out);
/* Device from_coo (graph.cpp:61-78): sort by (dst, src), reject ids out of
 * range (GF_ERR_GRAPH, *bad = input edge index) and duplicates (GF_ERR_GRAPH,
 * *bad = -2 - sorted position), build CSR and CSC (+ csc_edge_perm) bit-exact
 * with the reference.  d_src/d_dst are device int64 arrays of length e.
 * Outputs (device, caller-allocated, int64 like graphfuse::Graph):
 * row_ptr[n+1], col[e], csc_ptr[n+1], csc_row[e], csc_perm[e]. */
int gf_from_coo_device(int64_t n, int64_t e, const int64_t* d_src, const int64_t* d_dst,
                       int64_t* d_row_ptr, int64_t* d_col, int64_t* d_csc_ptr,
                       int64_t* d_csc_row, int64_t* d_csc_perm, int64_t* bad, void* stream);
/* Multi-CTA split of super rows / columns: a CTA-bucket row of degree d runs
 * on ceil(d / split_len) CTAs (slice states merged in slice order by the
 * last one).  Default split_len = max(cta_threshold, ceil(E / (148 * 4))) of
 * the graph's own edge count; a row-sharded graph takes the unsharded
 * graph's value here so its per-row reduction order, hence its results, stay
 * bitwise equal to 1 GPU.  Not concurrent with launches on the graph. */
int gf_graph_set_split_len(gf_graph_t g, int64_t split_len, void* stream);
int gf_graph_destroy(gf_graph_t g);
int gf_graph_get_info(gf_graph_t g, gf_graph_info* info);
/* Copy the device schedules to host (row_order[n], col_order[n]; int32). */
int gf_graph_get_schedule(gf_graph_t g, int32_t* row_order, int32_t* col_order);

/* ---- fused forward (replaces run_block_rows, engine.hpp:192-231) ----
 * One launch: SDDMM -> per-destination softmax -> SpMM; writes O and the
 * stats records only (no E x H tensor).  P (E x H, CSR order) is
 * materialised by a second recompute launch only when P != NULL (reference
 * ForwardContext::P). */
int gf_attn_fwd(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                const void* V, void* O, void* stats, void* P, void* stream);

/* ---- forward under an explicit fusion strategy (run_smmf / run_pmf /
 * run_unfused / run_feature_parallel_baseline, engine.hpp:292-329) ----
 * Same outputs as gf_attn_fwd (O, the softmax records, P when non-NULL) for
 * every strategy; they differ in launch structure and HBM traffic only.
 * PMF and unfused need E*H (unfused without P: 2*E*H) elements of scratch:
 * gf_attn_fwd_workspace reports the bytes; workspace == NULL makes the call
 * allocate (stream-ordered) and free it itself. */
int gf_attn_fwd_workspace(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy,
                          int32_t have_p, size_t* bytes);
int gf_attn_fwd_strategy(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy, const void* Q,
                         const void* K, const void* V, void* O, void* stats, void* P,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Device time of the strategy's forward on resident inputs: one warm-up call,
 * then `reps` calls bracketed by CUDA events on `stream`; *ms_out = mean ms
 * per forward.  Synchronises `stream`.  (The bench harness, run_benchmark,
 * reports this measured GPU time next to the reference's modelled counters.) */
int gf_time_fwd_strategy(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy, const void* Q,
                         const void* K, const void* V, void* O, void* stats, int32_t reps,
                         float* ms_out, void* stream);

/* ---- single-step operators (the unfused schedule's building blocks) ----
 * E x H edge tensors are CSR-ordered, head-minor ([e][h]).  Each call is
 * one kernel (two for spmm_backward / sddmm_backward) and moves its E x H
 * operands through HBM, as the reference's unfused counters model.
 * Ops that visit the CSC view need an unsharded graph. */
/* sddmm (kernels.hpp:18-47, 106-117): S[e,h] = scale <Q[src], K[dst]> (dot;
 * l2: on L2-normalised rows) or LeakyReLU(el[src] + er[dst]) (add). */
int gf_sddmm(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K, void* S,
             void* stream);
/* edge_softmax (kernels.hpp:65-82): per destination row and head. */
int gf_edge_softmax(gf_graph_t g, int32_t dtype, int32_t heads, const void* S, void* P,
                    void* stream);
/* spmm (kernels.hpp:85-102): O[v] = sum_{e in row v} P[e] V[src e] per head. */
int gf_spmm(gf_graph_t g, int32_t dtype, int32_t heads, int32_t head_dim, const void* P,
            const void* V, void* O, void* stream);
/* l2_normalize_rows (kernels.hpp:50-61) per head segment (x / max(||x||,
 * eps), eps > 0) and its backward (autograd.hpp:76-95).  X, Y, dY, dX:
 * n x (heads*head_dim). */
int gf_l2_normalize_rows(int32_t dtype, int64_t n, int32_t heads, int32_t head_dim, const void* X,
                         void* Y, double eps, void* stream);
int gf_l2_normalize_backward(int32_t dtype, int64_t n, int32_t heads, int32_t head_dim,
                             const void* X, const void* dY, void* dX, double eps, void* stream);
/* spmm_backward (autograd.hpp:33-58): dP[e] = <dO[dst], V[src]>,
 * dV[u] = sum over u's out-edges of P[e] dO[dst]. */
int gf_spmm_backward(gf_graph_t g, int32_t dtype, int32_t heads, int32_t head_dim, const void* P,
                     const void* V, const void* dO, void* dP, void* dV, void* stream);
/* softmax_backward (autograd.hpp:62-73): dS = P (dP - sum_row P dP). */
int gf_softmax_backward(gf_graph_t g, int32_t dtype, int32_t heads, const void* P, const void* dP,
                        void* dS, void* stream);
/* sddmm_backward (autograd.hpp:102-154): dot -> dQ (out-edges, K[dst]) and
 * dK (in-edges, Q[src]), through the L2 normalisation when desc->l2; add ->
 * del, der (N x H) with the LeakyReLU derivative (kink takes the slope). */
int gf_sddmm_backward(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                      const void* dS, void* dQ, void* dK, void* stream);

/* dense_oracle_forward (kernels.hpp:122-166), single head: the reference's
 * masked dense test oracle on the device.  S (n x n, caller-allocated,
 * row-major) gets S[v*n+u] = score of edge u -> v and 0 off the mask; O
 * (n x v_cols) = row softmax over the mask (u ascending) times V, densely.
 * desc: heads = 1, head_dim = Q/K width (1 for GF_ADD), scale / slope / l2 as
 * in SddmmKind.  coo_src/coo_dst: device int64 [e] (the Graph's COO).
 * n > 4096 -> GF_ERR_INVALID ("dense_oracle_forward: N > 4096"). */
int gf_dense_oracle_forward(int64_t n, int64_t e, const int64_t* coo_src, const int64_t* coo_dst,
                            const gf_attn_desc* desc, int64_t v_cols, const void* Q,
                            const void* K, const void* V, void* S, void* O, void* stream);

/* ---- recompute backward (replaces backward_values, autograd.hpp:158-170) ----
 * Pass A over CSR rows (dK or der, and delta into stats), pass B over CSC
 * columns (dQ or del, dV).  Attention is recomputed from the stats records;
 * no E x H tensor is read or written.  stats is read-write (delta). */
int gf_attn_bwd(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                const void* V, const void* O, void* stats, const void* dO, void* dQ, void* dK,
                void* dV, void* stream);
/* The two passes separately (same arguments; pass B reads the delta pass A
 * wrote).  Lets a caller time them apart or overlap pass B's inputs (e.g. an
 * all-gather of dO and the records in the row-sharded multi-GPU path). */
int gf_attn_bwd_rows(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                     const void* V, const void* O, void* stats, const void* dO, void* dK,
                     void* stream);
int gf_attn_bwd_cols(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                     const void* V, const void* stats, const void* dO, void* dQ, void* dV,
                     void* stream);

/* ---- dense projections (replaces matmul / matmul_at_b, models.hpp:58-86) ----
 * C[M x N] = A[M x K] * B[K x N]          (trans_a = 0)
 * C[M x N] = A[K x M]^T * B[K x N]        (trans_a = 1)
 * Row-major, fp32 or fp64; accumulate = 1 adds into C. */
int gf_gemm(int32_t dtype, int32_t trans_a, int64_t M, int64_t N, int64_t K, const void* A,
            const void* B, void* C, int32_t accumulate, void* stream);
/* Merge of source-phased forward partials (row-sharded overlap, SURVEY
 * §8(e)): part k is the forward over the in-edges whose sources lie in block
 * k (its sub-graph row pointer row_ptrs[k], normalised O_parts[k] rows x F,
 * records rec_parts[k] rows x H x 4).  Per (row, head): m = max m_k,
 * w_k = l_k e^(m_k - m), O = sum w_k O_k / sum w_k, record {m, log2 sum w_k,
 * aux}; delta untouched; parts empty in a row are skipped, rows empty in all
 * parts untouched.  1 <= parts <= 8, heads <= 32.  All arrays row-relative. */
int gf_attn_merge_parts(int32_t dtype, int64_t rows, int32_t heads, int32_t head_dim,
                        int32_t parts, const int32_t* const* row_ptrs, const void* const* O_parts,
                        const void* const* rec_parts, void* O, void* rec, void* stream);

/* Projection fused with its all-gather: C = A·B (fp32,
 * 3xTF32 tcgen05, A M x K, B K x N row-major) stored by the TMA epilogue to
 * n_dst (1..8) row-major M x N destinations — dst[0] local, dst[1..] the
 * same rows of the peers' tables through peer-mapped (NVLink) addresses —
 * tile by tile.  Requires K % 4 == 0, N % 32 == 0, 16 B aligned pointers.
 * Replaces models.hpp:116-125's projections + the row all-gather. */
int gf_gemm_bcast(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* A, const void* B,
                  void* const* dst, int32_t n_dst, void* stream);
/* C = A·B (fp32, 3xTF32 tcgen05, TMA epilogue) with column block j (N / n_dst
 * columns, a multiple of 32) stored to dst[j] (row-major M x N / n_dst): the
 * GT / AGNN projections X·[W_q | W_k | W_v] as one GEMM writing Q, K, V into
 * their own tables (models.hpp:116-125).  16 B aligned, K % 4 == 0. */
int gf_gemm_split(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* A, const void* B,
                  void* const* dst, int32_t n_dst, void* stream);
/* C = A·B (fp32, 3xTF32 tcgen05, TMA epilogue) with column block j (N / n_dst
 * columns, a multiple of 32) stored to dst[j] (row-major M x N / n_dst): the
 * GT / AGNN projections X·[W_q | W_k | W_v] as one GEMM writing Q, K, V into
 * their own tables (models.hpp:116-125).  16 B aligned, K % 4 == 0. */
int gf_gemm_split(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* A, const void* B,
                  void* const* dst, int32_t n_dst, void* stream);
/* GAT attention logits: el[n,h] = sum_d Hf[n,h,d] a_l[h,d]; er likewise. */
int gf_gat_logits(int32_t dtype, int64_t n, int32_t H, int32_t D, const void* Hf, const void* a_l,
                  const void* a_r, void* el, void* er, void* stream);
/* GAT fan-in (models.hpp:143-148): dH = dV + del (x) a_l + der (x) a_r, and
 * da_l[h,d] = sum_n Hf[n,h,d] del[n,h], da_r likewise. */
int gf_gat_fanin(int32_t dtype, int64_t n, int32_t H, int32_t D, const void* Hf, const void* a_l,
                 const void* a_r, const void* dV, const void* del, const void* der, void* dH,
                 void* da_l, void* da_r, void* stream);

/* ---- synthetic graphs on the device ----
 * The reference's generators' distributions (graph.cpp:127-185), drawn with
 * counter-based hashing + radix-sort dedup instead of a sequential
 * mt19937_64 rejection loop: deterministic per seed, NOT the reference's
 * exact edge sequence.  Output: device int64 COO (src, dst) for
 * gf_from_coo_device; *e_out = edges written.
 *   random     : exactly round(n*avg_degree) distinct uniform edges
 *   super_node : node 0 gets exactly hub_degree distinct in-neighbours, the
 *                rest (max(hub, round(n*avg)) edges in total) uniform distinct
 *                edges with destinations != 0
 *   power_law  : row r of deg_r = round(max_degree (r+1)^-exponent) is a
 *                hashed node id, sources uniform, duplicate sources dropped
 *                (capacity >= sum deg_r)
 *   molecules  : `mols` disjoint blocks of `atoms` ids (the batch_graphs
 *                layout, graph.cpp:104-118), each a random spanning tree plus
 *                `rings` extra bonds, both directions, no self-loops or
 *                duplicates (capacity >= 2 mols (atoms - 1 + rings)) */
int gf_gen_random_device(int64_t n, double avg_degree, uint64_t seed, int64_t* src, int64_t* dst,
                         int64_t* e_out, void* stream);
int gf_gen_super_node_device(int64_t n, double avg_degree, int64_t hub_degree, uint64_t seed,
                             int64_t* src, int64_t* dst, int64_t* e_out, void* stream);
int gf_gen_power_law_device(int64_t n, int64_t max_degree, double exponent, uint64_t seed,
                            int64_t capacity, int64_t* src, int64_t* dst, int64_t* e_out,
                            void* stream);
int gf_gen_molecules_device(int64_t mols, int64_t atoms, int64_t rings, uint64_t seed,
                            int64_t capacity, int64_t* src, int64_t* dst, int64_t* e_out,
                            void* stream);

/* ---- device-wide state (opt-in; the library never changes it on its own) ----
 * gf_l2_persist(bytes): set cudaLimitPersistingL2CacheSize of the current
 * device to min(bytes, device max).  The kernels tag the gathered node
 * tables L2::evict_last, which keeps them resident only while a set-aside
 * exists (C4: +2-3 %).  bytes = 0 first demotes every persisting line
 * (cudaCtxResetPersistingL2Cache) and then removes the set-aside.
 * GF_L2_SETASIDE=<MiB> in the environment opts in at the first attention
 * call instead.  gf_l2_persist_get reads the current limit.
 * gf_l2_reset_persisting(): demote every persisting line to normal (e.g.
 * before a cold-L2 timing step), keeping the set-aside.
 * gf_scratch_trim(): synchronise the device and release the stream-ordered
 * scratch the library caches in its private memory pool. */
int gf_l2_persist(size_t bytes);
int gf_l2_persist_get(size_t* bytes);
int gf_l2_reset_persisting(void);
int gf_scratch_trim(void);

/* ---- measured counters (CUPTI range profiler; libcupti loaded on demand) ----
 * Runs fn(user) inside one profiled range, once per counter pass (user
 * replay; byte counters need one), with prep(user) (nullable) before each
 * pass outside the range, synchronising the device after each; evaluates the
 * n_metrics (1..16) Nsight-Compute-style metric names (e.g.
 * "dram__bytes_read.sum", "dram__bytes_write.sum",
 * "l1tex__m_xbar2l1tex_read_bytes.sum") into values.  GF_ERR_UNSUPPORTED
 * without libcupti or without profiling permission.  Not for timing runs. */
int gf_measure_metrics(void (*prep)(void*), void (*fn)(void*), void* user,
                       const char* const* metrics, int32_t n_metrics, double* values);

/* ---- diagnostics ----
 * Measured gather bandwidth (GB/s) of rows of row_bytes (32..1024, lanes read
 * consecutive 32 B chunks with 256-bit non-coherent loads) chosen in hashed
 * order from a footprint_bytes buffer, every SM, after a warm-up pass: with
 * an L2-resident footprint, the roofline denominator for the gather kernels. */
int gf_measure_l2_gather(size_t footprint_bytes, int32_t row_bytes, int32_t iters,
                         double* gbs_out, void* stream);
/* Design probe (profiles/r2/ab_r2_passb_alternatives.txt): mean ms of a
 * scatter over the CSC edges of a device graph's arrays into table[v][0..7]
 * (mode 0 red.add.f32, 1 red.add.v4.f32, 2 st.f32, 3 ld.f32, 4 red.add.u64),
 * `iters` launches after a warm-up. */
int gf_probe_scatter(int64_t n, const int32_t* csc_ptr, const int32_t* csc_row, float* table,
                     int32_t mode, int32_t iters, float* ms_out, void* stream);
/* The L2 evict_last policy word the backward passes receive in their argument
 * block (host_word, a compile-time constant) and the word createpolicy
 * produces on the device (device_word); the two must agree. */
int gf_l2_policy_word(uint64_t* device_word, uint64_t* host_word);

#ifdef __cplusplus
}
#endif
#endif /* GF_CUDA_H */

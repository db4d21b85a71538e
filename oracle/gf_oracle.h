/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 fused AT-GNN path.
 *
 * Plain-C restatement of the reference algorithm (arxiv/paper_2411_16127,
 * `graphfuse`, /root/reference/proj).  Each function cites the reference
 * file:line it restates.  Parity of this restatement is PINNED against the
 * reference itself (oracle/_ref/libgfref.so, built from the reference sources
 * by oracle/Makefile) and against golden vectors in tests/golden/ produced by
 * scripts/make_golden.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never does.
 *
 * Layout (multi-head; the reference is single-head, and is
 * applied per head h to column slices):
 *   dot: Q, K are N x (H*D) row-major; add (GAT): Q=el, K=er are N x H.
 *   V, O, dO, dV are N x (H*D).  P (optional) is E x H in CSR edge order.
 *   lse (optional) is N x H: zmax + log(zsum) per destination row and head.
 */
#ifndef GF_ORACLE_H
#define GF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* graph.cpp:61-78 (from_coo) + graph.cpp:25-57 (build_from_sorted).
 * Returns 0, 1 (id out of range, *bad = edge index) or 2 (duplicate). */
int gfo_from_coo(int64_t n, int64_t e, const int64_t* src, const int64_t* dst, int64_t* row_ptr,
                 int64_t* col, int64_t* csc_ptr, int64_t* csc_row, int64_t* csc_perm,
                 int64_t* bad);

/* Degree-bucket schedule (no reference counterpart: restates the B200
 * scheduler's definition so the device schedule can be checked bit-exactly).
 * order = rows stably sorted by degree descending; n_cta = #rows with
 * degree >= cta_threshold (they lead the order); n_empty = #rows of degree 0
 * (they trail it); n_small = #rows of degree 1..GFO_SMALL_DEGREE below the
 * CTA threshold (just before the empty ones). */
#define GFO_SMALL_DEGREE 8 /* rows of degree 1..8 form the packed (sub-warp) bucket */
void gfo_schedule(int64_t n, const int64_t* ptr, int64_t cta_threshold, int32_t* order,
                  int64_t* n_cta, int64_t* n_empty, int64_t* n_small);

/* engine.hpp:192-231 (run_block_rows) + kernels.hpp:50-61 (l2_normalize_rows)
 * per head.  variant: 0 dot, 1 add. */
int gfo_forward_f32(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col, int H,
                    int D, int variant, int l2, double scale, double slope, const float* Q,
                    const float* K, const float* V, float* O, float* P, float* lse);
int gfo_forward_f64(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col, int H,
                    int D, int variant, int l2, double scale, double slope, const double* Q,
                    const double* K, const double* V, double* O, double* P, double* lse);

/* autograd.hpp:158-170 (backward_values) on P = edge_softmax(sddmm(Q,K))
 * exactly as the Python binding rebuilds it (module.cpp:128). */
int gfo_backward_f32(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col,
                     const int64_t* csc_ptr, const int64_t* csc_row, const int64_t* csc_perm,
                     int H, int D, int variant, int l2, double scale, double slope,
                     const float* Q, const float* K, const float* V, const float* dO, float* dQ,
                     float* dK, float* dV);
int gfo_backward_f64(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col,
                     const int64_t* csc_ptr, const int64_t* csc_row, const int64_t* csc_perm,
                     int H, int D, int variant, int l2, double scale, double slope,
                     const double* Q, const double* K, const double* V, const double* dO,
                     double* dQ, double* dK, double* dV);

/* Same plus the edge gradients dP and dS (E x H, CSR order; nullable). */
int gfo_backward2_f32(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col,
                      const int64_t* csc_ptr, const int64_t* csc_row, const int64_t* csc_perm,
                      int H, int D, int variant, int l2, double scale, double slope,
                      const float* Q, const float* K, const float* V, const float* dO, float* dQ,
                      float* dK, float* dV, float* dP, float* dS);
int gfo_backward2_f64(int64_t n, int64_t e, const int64_t* row_ptr, const int64_t* col,
                      const int64_t* csc_ptr, const int64_t* csc_row, const int64_t* csc_perm,
                      int H, int D, int variant, int l2, double scale, double slope,
                      const double* Q, const double* K, const double* V, const double* dO,
                      double* dQ, double* dK, double* dV, double* dP, double* dS);

#ifdef __cplusplus
}
#endif
#endif

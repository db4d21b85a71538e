/* TEST INFRASTRUCTURE ONLY — see gf_oracle.h for scope and pinning. */
#include "gf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- graph -- */

/* graph.cpp:61-78: validate ids in input order (67-69), order edges by
 * (dst, src) (72), reject duplicates (73-76).  The ordering is done here with
 * two stable counting passes (src, then dst) — same result as the reference's
 * comparison sort.  graph.cpp:31-41 CSR by counting; graph.cpp:43-55 CSC by a
 * stable bucket scatter over CSR order, so each column is sorted by dst. */
int gfo_from_coo(int64_t n, int64_t e, const int64_t* src, const int64_t* dst, int64_t* row_ptr,
                 int64_t* col, int64_t* csc_ptr, int64_t* csc_row, int64_t* csc_perm,
                 int64_t* bad) {
  for (int64_t i = 0; i < e; ++i) {
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) {
      if (bad) *bad = i;
      return 1;
    }
  }
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(e > 0 ? e : 1));
  /* pass 1: stable by src */
  for (int64_t i = 0; i < e; ++i) cnt[src[i] + 1]++;
  for (int64_t u = 0; u < n; ++u) cnt[u + 1] += cnt[u];
  for (int64_t i = 0; i < e; ++i) tmp[cnt[src[i]]++] = i;
  /* pass 2: stable by dst -> (dst, src) order; CSR row pointer falls out */
  memset(row_ptr, 0, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < e; ++i) row_ptr[dst[i] + 1]++;
  for (int64_t v = 0; v < n; ++v) row_ptr[v + 1] += row_ptr[v];
  memcpy(cnt, row_ptr, sizeof(int64_t) * ((size_t)n + 1));
  int64_t* coo_dst = (int64_t*)malloc(sizeof(int64_t) * (size_t)(e > 0 ? e : 1));
  for (int64_t k = 0; k < e; ++k) {
    int64_t i = tmp[k];
    int64_t slot = cnt[dst[i]]++;
    col[slot] = src[i];
    coo_dst[slot] = dst[i];
  }
  for (int64_t i = 1; i < e; ++i) {
    if (coo_dst[i] == coo_dst[i - 1] && col[i] == col[i - 1]) {
      if (bad) *bad = i;
      free(cnt), free(tmp), free(coo_dst);
      return 2;
    }
  }
  memset(csc_ptr, 0, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < e; ++i) csc_ptr[col[i] + 1]++;
  for (int64_t u = 0; u < n; ++u) csc_ptr[u + 1] += csc_ptr[u];
  memcpy(cnt, csc_ptr, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < e; ++i) {
    int64_t slot = cnt[col[i]]++;
    csc_row[slot] = coo_dst[i];
    csc_perm[slot] = i;
  }
  free(cnt), free(tmp), free(coo_dst);
  return 0;
}

/* ------------------------------------------------------------- schedule -- */

void gfo_schedule(int64_t n, const int64_t* ptr, int64_t cta_threshold, int32_t* order,
                  int64_t* n_cta, int64_t* n_empty, int64_t* n_small) {
  /* Stable sort by degree descending = counting sort over distinct degrees.
   * Degrees are bounded by E, so use a sort on (deg desc, row asc) pairs via
   * a simple merge sort of row indices keyed by degree. */
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) {
        int64_t da = ptr[idx[a] + 1] - ptr[idx[a]], db = ptr[idx[b] + 1] - ptr[idx[b]];
        buf[o++] = (db > da) ? idx[b++] : idx[a++]; /* ties keep left (stable) */
      }
      while (a < mid) buf[o++] = idx[a++];
      while (b < hi) buf[o++] = idx[b++];
    }
    int64_t* t = idx;
    idx = buf;
    buf = t;
  }
  int64_t c = 0, z = 0, sm = 0;
  for (int64_t i = 0; i < n; ++i) {
    order[i] = (int32_t)idx[i];
    int64_t d = ptr[idx[i] + 1] - ptr[idx[i]];
    if (d >= cta_threshold && d > 0) ++c;
    if (d == 0) ++z;
    if (d >= 1 && d <= GFO_SMALL_DEGREE && d < cta_threshold) ++sm;
  }
  *n_cta = c;
  *n_empty = z;
  if (n_small) *n_small = sm;
  free(idx);
  free(buf);
}

/* --------------------------------------------------- forward / backward -- */

#define GFO_T float
#define GFO_SUFFIX f32
#include "gf_oracle_impl.inc"
#undef GFO_T
#undef GFO_SUFFIX

#define GFO_T double
#define GFO_SUFFIX f64
#include "gf_oracle_impl.inc"
#undef GFO_T
#undef GFO_SUFFIX

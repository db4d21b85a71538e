// Device topology and the bi-level degree-bucket scheduler.
//
//  * gf_graph_create*: int32 CSR (destination rows) + CSC (source columns)
//    resident in HBM, plus two schedules: rows (forward, backward pass A) and
//    columns (backward pass B) stably sorted by degree descending with
//    cub::DeviceRadixSort (LSD radix sort is stable, so ties keep ascending
//    node id — the CPU restatement gfo_schedule defines the same order and
//    tests compare them bit-exactly).  Bucket counts: rows with degree >=
//    cta_threshold (CTA / edge-split bucket, they lead the order) and empty
//    rows (they trail it); everything between is the warp-per-row bucket.
//  * gf_from_coo_device: the reference's from_coo (graph.cpp:61-78) on the
//    GPU: id validation, (dst,src) radix sort, duplicate rejection, CSR by
//    segment offsets and the CSC transpose (+ csc_edge_perm) by a second
//    (src,dst) sort — bit-exact with graph.cpp:25-57.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {

namespace {

__global__ void degrees_kernel(const int32_t* __restrict__ ptr, int n, int32_t* __restrict__ deg,
                               int32_t* __restrict__ ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    deg[i] = ptr[i + 1] - ptr[i];
    ids[i] = i;
  }
}

// stats[0] = max degree, stats[1] = #(deg >= thr), stats[2] = #(deg == 0),
// stats[3] = #(1 <= deg <= kSmallDegree, deg < thr)
__global__ void degree_stats_kernel(const int32_t* __restrict__ deg, int n, int thr,
                                    int32_t* __restrict__ stats) {
  int mx = 0, big = 0, zero = 0, small = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = deg[i];
    mx = max(mx, d);
    big += (d >= thr && d > 0);
    zero += (d == 0);
    small += (d >= 1 && d <= kSmallDegree && d < thr);
  }
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    big += __shfl_xor_sync(kFull, big, o);
    zero += __shfl_xor_sync(kFull, zero, o);
    small += __shfl_xor_sync(kFull, small, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(stats + 0, mx);
    atomicAdd(stats + 1, big);
    atomicAdd(stats + 2, zero);
    atomicAdd(stats + 3, small);
  }
}

int bits_for(long long x) {
  int b = 1;
  while ((1LL << b) <= x) ++b;
  return b;
}

// Degree-descending stable order of [0, n) for a pointer array.
int build_schedule(const int32_t* d_ptr, int n, int thr, int32_t* d_order, int32_t& n_cta,
                   int32_t& n_empty, int32_t& n_small, int64_t& max_deg, cudaStream_t s) {
  if (n == 0) {
    n_cta = n_empty = n_small = 0;
    max_deg = 0;
    return GF_OK;
  }
  int32_t *deg = nullptr, *ids = nullptr, *deg_sorted = nullptr, *stats = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&deg, sizeof(int32_t) * n, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&ids, sizeof(int32_t) * n, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&deg_sorted, sizeof(int32_t) * n, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&stats, sizeof(int32_t) * 4, s));
  GF_CHECK_CUDA(cudaMemsetAsync(stats, 0, sizeof(int32_t) * 4, s));
  degrees_kernel<<<(n + 255) / 256, 256, 0, s>>>(d_ptr, n, deg, ids);
  GF_CHECK_LAUNCH("degrees_kernel");
  degree_stats_kernel<<<min(1024, (n + 255) / 256), 256, 0, s>>>(deg, n, thr, stats);
  GF_CHECK_LAUNCH("degree_stats_kernel");
  int32_t h[4];
  GF_CHECK_CUDA(cudaMemcpyAsync(h, stats, sizeof(h), cudaMemcpyDeviceToHost, s));
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  max_deg = h[0];
  n_cta = h[1];
  n_empty = h[2];
  n_small = h[3];
  const int end_bit = bits_for(h[0]);
  size_t tmp_bytes = 0;
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, deg, deg_sorted,
                                                           ids, d_order, n, 0, end_bit, s));
  void* tmp = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, tmp_bytes, s));
  GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, deg, deg_sorted, ids,
                                                           d_order, n, 0, end_bit, s));
  GF_CHECK_LAUNCH("radix sort");
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(deg, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(deg_sorted, s);
  cudaFreeAsync(stats, s);
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

__global__ void sched_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ ptr,
                             int n, int4* __restrict__ sched) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = order[i];
    sched[i] = make_int4(v, ptr[v], ptr[v + 1], 0);
  }
}

int build_sched(const int32_t* order, const int32_t* ptr, int n, int4** out, cudaStream_t s) {
  GF_CHECK_CUDA(cudaMalloc(out, sizeof(int4) * (n > 0 ? n : 1)));
  if (n == 0) return GF_OK;
  sched_kernel<<<std::min(4096, (n + 255) / 256), 256, 0, s>>>(order, ptr, n, *out);
  GF_CHECK_LAUNCH("sched_kernel");
  return GF_OK;
}

// CTA-bucket block table of one pass: the first n_cta schedule slots are the
// CTA rows (degree-descending); a row of degree d gets ceil(d / split_len)
// blocks {slot, slice, slices, first partial}; single-slice rows carry -1.
int build_cta_table(const int4* sched, int n_cta, int64_t len, int4** tab, int32_t& blocks,
                    int32_t& parts, cudaStream_t s) {
  blocks = parts = 0;
  cudaFree(*tab);
  *tab = nullptr;
  if (n_cta == 0) return GF_OK;
  std::vector<int4> h(static_cast<size_t>(n_cta));
  GF_CHECK_CUDA(cudaMemcpyAsync(h.data(), sched, sizeof(int4) * n_cta, cudaMemcpyDeviceToHost, s));
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  std::vector<int4> t;
  t.reserve(static_cast<size_t>(n_cta));
  for (int r = 0; r < n_cta; ++r) {
    const int64_t d = static_cast<int64_t>(h[r].z) - h[r].y;
    const int ns = static_cast<int>(std::max<int64_t>(1, (d + len - 1) / len));
    const int base = ns > 1 ? parts : -1;
    for (int k = 0; k < ns; ++k) t.push_back(make_int4(r, k, ns, base));
    if (ns > 1) parts += ns;
  }
  blocks = static_cast<int32_t>(t.size());
  GF_CHECK_CUDA(cudaMalloc(tab, sizeof(int4) * t.size()));
  GF_CHECK_CUDA(cudaMemcpyAsync(*tab, t.data(), sizeof(int4) * t.size(), cudaMemcpyHostToDevice, s));
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

int finish_graph(DevGraph* g, int thr, cudaStream_t s) {
  g->cta_threshold = thr > 0 ? thr : auto_cta_threshold(std::max<int64_t>(g->e, g->e_csc));
  GF_CHECK_CUDA(cudaGetDevice(&g->device));
  GF_CHECK_CUDA(cudaMalloc(&g->row_order, sizeof(int32_t) * (g->n > 0 ? g->n : 1)));
  GF_CHECK_CUDA(cudaMalloc(&g->col_order, sizeof(int32_t) * (g->n > 0 ? g->n : 1)));
  int rc = build_schedule(g->row_ptr, g->n, g->cta_threshold, g->row_order, g->n_cta_rows,
                          g->n_empty_rows, g->n_small_rows, g->max_in, s);
  if (rc) return rc;
  rc = build_schedule(g->csc_ptr, g->n, g->cta_threshold, g->col_order, g->n_cta_cols,
                      g->n_empty_cols, g->n_small_cols, g->max_out, s);
  if (rc) return rc;
  if ((rc = build_sched(g->row_order, g->row_ptr, g->n, &g->row_sched, s))) return rc;
  if ((rc = build_sched(g->col_order, g->csc_ptr, g->n, &g->col_sched, s))) return rc;
  if ((rc = build_cta_table(g->row_sched, g->n_cta_rows, split_len(g->e, g->cta_threshold),
                            &g->row_cta, g->row_cta_blocks, g->row_parts, s)))
    return rc;
  if ((rc = build_cta_table(g->col_sched, g->n_cta_cols, split_len(g->e_csc, g->cta_threshold),
                            &g->col_cta, g->col_cta_blocks, g->col_parts, s)))
    return rc;
  GF_CHECK_CUDA(cudaStreamSynchronize(s));
  return GF_OK;
}

void free_graph(DevGraph* g) {
  if (!g) return;
  cudaFree(g->row_ptr);
  cudaFree(g->col);
  cudaFree(g->csc_ptr);
  cudaFree(g->csc_row);
  cudaFree(g->row_order);
  cudaFree(g->col_order);
  cudaFree(g->row_sched);
  cudaFree(g->col_sched);
  cudaFree(g->row_cta);
  cudaFree(g->col_cta);
  cudaFree(g->coo_dst);
  cudaFree(g->csc_perm);
  delete g;
}

// ------------------------------------------------------- device from_coo --
__global__ void coo_check_pack(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                               int64_t e, int64_t n, int b, uint64_t* __restrict__ k_ds,
                               unsigned long long* __restrict__ bad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t u = src[i], v = dst[i];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      atomicMin(bad, static_cast<unsigned long long>(i));
      k_ds[i] = 0;
    } else {
      k_ds[i] = (static_cast<uint64_t>(v) << b) | static_cast<uint64_t>(u);
    }
  }
}

// Unpack sorted keys into (major, minor) arrays, flag duplicates, and write
// the segment pointer of the major index (ptr[x] = first position >= x).
__global__ void unpack_sorted(const uint64_t* __restrict__ keys, int64_t e, int64_t n, int b,
                              int64_t* __restrict__ minor, int64_t* __restrict__ ptr,
                              unsigned long long* __restrict__ dup) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cur = i < e ? static_cast<int64_t>(keys[i] >> b) : n;
    const int64_t prev = i > 0 ? static_cast<int64_t>(keys[i - 1] >> b) : -1;
    if (i < e) {
      minor[i] = static_cast<int64_t>(keys[i] & mask);
      if (i > 0 && keys[i] == keys[i - 1]) atomicMin(dup, static_cast<unsigned long long>(i));
    }
    for (int64_t x = prev + 1; x <= cur; ++x) ptr[x] = i;
  }
}

// CSR-sorted keys (v, u) -> swapped keys (u, v) carrying their CSR edge id:
// sorting these pairs yields the CSC order and, in the values, csc_edge_perm
// (CSC slot -> CSR edge id) with no search.
__global__ void swap_with_ids(const uint64_t* __restrict__ k_ds, int64_t e, int b,
                              uint64_t* __restrict__ k_sd, int32_t* __restrict__ ids) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = k_ds[i];
    k_sd[i] = ((k & mask) << b) | (k >> b);
    ids[i] = static_cast<int32_t>(i);
  }
}

__global__ void widen_ids(const int32_t* __restrict__ ids, int64_t e, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = ids[i];
}
}  // namespace

}  // namespace gfb

using gfb::DevGraph;


extern "C" int gf_graph_create_split(int64_t n, int64_t e_csr, const int32_t* d_row_ptr,
                                     const int32_t* d_col, int64_t e_csc,
                                     const int32_t* d_csc_ptr, const int32_t* d_csc_row,
                                     int32_t cta_threshold, int32_t flags, void* stream,
                                     gf_graph_t* out) {
  constexpr int64_t kMax = (1LL << 31) - 1;
  if (!out || n < 0 || e_csr < 0 || e_csc < 0 || n >= kMax || e_csr >= kMax || e_csc >= kMax) {
    gfb::set_error("gf_graph_create: invalid sizes (int32 node/edge ids required)");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  auto* g = new gf_graph_s();
  g->n = static_cast<int32_t>(n);
  g->e = static_cast<int32_t>(e_csr);
  g->e_csc = static_cast<int32_t>(e_csc);
  g->skip_empty = (flags & GF_GRAPH_SKIP_EMPTY) != 0;
  const size_t np = sizeof(int32_t) * (n + 1);
  const size_t er = sizeof(int32_t) * (e_csr > 0 ? e_csr : 1);
  const size_t ec = sizeof(int32_t) * (e_csc > 0 ? e_csc : 1);
  auto fail = [&](int rc) {
    gfb::free_graph(g);
    return rc;
  };
  if (cudaMalloc(&g->row_ptr, np) || cudaMalloc(&g->col, er) || cudaMalloc(&g->csc_ptr, np) ||
      cudaMalloc(&g->csc_row, ec)) {
    gfb::set_error("gf_graph_create: cudaMalloc failed");
    return fail(GF_ERR_CUDA);
  }
  if (cudaMemcpyAsync(g->row_ptr, d_row_ptr, np, cudaMemcpyDeviceToDevice, s) ||
      cudaMemcpyAsync(g->csc_ptr, d_csc_ptr, np, cudaMemcpyDeviceToDevice, s) ||
      (e_csr > 0 &&
       cudaMemcpyAsync(g->col, d_col, sizeof(int32_t) * e_csr, cudaMemcpyDeviceToDevice, s)) ||
      (e_csc > 0 && cudaMemcpyAsync(g->csc_row, d_csc_row, sizeof(int32_t) * e_csc,
                                    cudaMemcpyDeviceToDevice, s))) {
    gfb::set_error("gf_graph_create: copy failed");
    return fail(GF_ERR_CUDA);
  }
  int rc = gfb::finish_graph(g, cta_threshold, s);
  if (rc) return fail(rc);
  *out = g;
  return GF_OK;
}

extern "C" int gf_graph_create_device(int64_t n, int64_t e, const int32_t* d_row_ptr,
                                      const int32_t* d_col, const int32_t* d_csc_ptr,
                                      const int32_t* d_csc_row, int32_t cta_threshold,
                                      void* stream, gf_graph_t* out) {
  return gf_graph_create_split(n, e, d_row_ptr, d_col, e, d_csc_ptr, d_csc_row, cta_threshold, 0,
                               stream, out);
}

extern "C" int gf_graph_create(int64_t n, int64_t e, const int64_t* row_ptr,
                               const int64_t* col, const int64_t* csc_ptr,
                               const int64_t* csc_row, int32_t cta_threshold, void* stream,
                               gf_graph_t* out) {
  if (!out || n < 0 || e < 0 || n >= (1LL << 31) - 1 || e >= (1LL << 31) - 1 ||
      (n > 0 && (!row_ptr || !csc_ptr)) || (e > 0 && (!col || !csc_row))) {
    gfb::set_error("gf_graph_create: invalid arguments (int32 node/edge ids required)");
    return GF_ERR_INVALID;
  }
  if (row_ptr && (row_ptr[0] != 0 || row_ptr[n] != e)) {
    gfb::set_error("gf_graph_create: csr_row_ptr must start at 0 and end at num_edges");
    return GF_ERR_GRAPH;
  }
  auto s = static_cast<cudaStream_t>(stream);
  std::vector<int32_t> h_rp(n + 1), h_cp(n + 1), h_col(e > 0 ? e : 1), h_cr(e > 0 ? e : 1);
  for (int64_t i = 0; i <= n; ++i) {
    h_rp[i] = static_cast<int32_t>(row_ptr ? row_ptr[i] : 0);
    h_cp[i] = static_cast<int32_t>(csc_ptr ? csc_ptr[i] : 0);
  }
  for (int64_t i = 0; i < e; ++i) {
    h_col[i] = static_cast<int32_t>(col[i]);
    h_cr[i] = static_cast<int32_t>(csc_row[i]);
  }
  int32_t *d_rp = nullptr, *d_cp = nullptr, *d_col = nullptr, *d_cr = nullptr;
  const size_t np = sizeof(int32_t) * (n + 1), ep = sizeof(int32_t) * (e > 0 ? e : 1);
  if (cudaMalloc(&d_rp, np) || cudaMalloc(&d_cp, np) || cudaMalloc(&d_col, ep) ||
      cudaMalloc(&d_cr, ep)) {
    cudaFree(d_rp), cudaFree(d_cp), cudaFree(d_col), cudaFree(d_cr);
    gfb::set_error("gf_graph_create: cudaMalloc failed");
    return GF_ERR_CUDA;
  }
  cudaMemcpyAsync(d_rp, h_rp.data(), np, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_cp, h_cp.data(), np, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_col, h_col.data(), ep, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_cr, h_cr.data(), ep, cudaMemcpyHostToDevice, s);
  int rc = gf_graph_create_device(n, e, d_rp, d_col, d_cp, d_cr, cta_threshold, stream, out);
  cudaStreamSynchronize(s);
  cudaFree(d_rp), cudaFree(d_cp), cudaFree(d_col), cudaFree(d_cr);
  return rc;
}

extern "C" int gf_graph_destroy(gf_graph_t g) {
  gfb::free_graph(g);
  return GF_OK;
}

extern "C" int gf_graph_get_info(gf_graph_t g, gf_graph_info* info) {
  if (!g || !info) {
    gfb::set_error("gf_graph_get_info: null argument");
    return GF_ERR_INVALID;
  }
  info->num_nodes = g->n;
  info->num_edges = g->e;
  info->max_in_degree = g->max_in;
  info->max_out_degree = g->max_out;
  info->cta_threshold = g->cta_threshold;
  info->n_cta_rows = g->n_cta_rows;
  info->n_empty_rows = g->n_empty_rows;
  info->n_cta_cols = g->n_cta_cols;
  info->n_empty_cols = g->n_empty_cols;
  info->device = g->device;
  info->n_small_rows = g->n_small_rows;
  info->n_small_cols = g->n_small_cols;
  info->cta_blocks_rows = g->row_cta_blocks;
  info->cta_blocks_cols = g->col_cta_blocks;
  return GF_OK;
}

extern "C" int gf_graph_get_schedule(gf_graph_t g, int32_t* row_order, int32_t* col_order) {
  if (!g) {
    gfb::set_error("gf_graph_get_schedule: null graph");
    return GF_ERR_INVALID;
  }
  if (g->n == 0) return GF_OK;
  if (row_order)
    GF_CHECK_CUDA(cudaMemcpy(row_order, g->row_order, sizeof(int32_t) * g->n,
                             cudaMemcpyDeviceToHost));
  if (col_order)
    GF_CHECK_CUDA(cudaMemcpy(col_order, g->col_order, sizeof(int32_t) * g->n,
                             cudaMemcpyDeviceToHost));
  return GF_OK;
}

extern "C" int gf_from_coo_device(int64_t n, int64_t e, const int64_t* d_src,
                                  const int64_t* d_dst, int64_t* d_row_ptr, int64_t* d_col,
                                  int64_t* d_csc_ptr, int64_t* d_csc_row, int64_t* d_csc_perm,
                                  int64_t* bad, void* stream) {
  using namespace gfb;
  if (n < 0 || e < 0 || n >= (1LL << 31) || e >= (1LL << 31)) {
    set_error("gf_from_coo_device: invalid sizes (node and edge counts must fit int32)");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  if (bad) *bad = -1;
  const int b = bits_for(n > 0 ? n - 1 : 0);
  const int grid = static_cast<int>(std::min<int64_t>(4096, (e + 255) / 256 + 1));
  uint64_t *k_ds = nullptr, *k_sd = nullptr, *k_ds_s = nullptr, *k_sd_s = nullptr;
  unsigned long long* flags = nullptr;
  const size_t eb = sizeof(uint64_t) * (e > 0 ? e : 1);
  GF_CHECK_CUDA(gfb::scratch_alloc(&k_ds, eb, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&k_sd, eb, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&k_ds_s, eb, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&k_sd_s, eb, s));
  GF_CHECK_CUDA(gfb::scratch_alloc(&flags, 2 * sizeof(unsigned long long), s));
  GF_CHECK_CUDA(cudaMemsetAsync(flags, 0xff, 2 * sizeof(unsigned long long), s));
  int rc = GF_OK;
  unsigned long long hflags[2] = {~0ull, ~0ull};
  if (e > 0) {
    coo_check_pack<<<grid, 256, 0, s>>>(d_src, d_dst, e, n, b, k_ds, flags);
    GF_CHECK_LAUNCH("coo_check_pack");
    int32_t *ids = nullptr, *ids_s = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&ids, sizeof(int32_t) * e, s));
    GF_CHECK_CUDA(gfb::scratch_alloc(&ids_s, sizeof(int32_t) * e, s));
    size_t tk = 0, tp = 0;
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tk, k_ds, k_ds_s, e, 0, 2 * b, s));
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tp, k_sd, k_sd_s, ids, ids_s, e, 0,
                                                  2 * b, s));
    const size_t tb = std::max(tk, tp);
    void* tmp = nullptr;
    GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, tb, s));
    size_t t = tb;
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t, k_ds, k_ds_s, e, 0, 2 * b, s));
    swap_with_ids<<<grid, 256, 0, s>>>(k_ds_s, e, b, k_sd, ids);
    GF_CHECK_LAUNCH("swap_with_ids");
    t = tb;
    GF_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, k_sd, k_sd_s, ids, ids_s, e, 0, 2 * b, s));
    cudaFreeAsync(tmp, s);
    // csc_edge_perm (graph.cpp:43-55's stable bucket scatter, as a pair sort)
    widen_ids<<<grid, 256, 0, s>>>(ids_s, e, d_csc_perm);
    GF_CHECK_LAUNCH("widen_ids");
    cudaFreeAsync(ids, s);
    cudaFreeAsync(ids_s, s);
    unpack_sorted<<<grid, 256, 0, s>>>(k_ds_s, e, n, b, d_col, d_row_ptr, flags + 1);
    GF_CHECK_LAUNCH("unpack_sorted csr");
    unpack_sorted<<<grid, 256, 0, s>>>(k_sd_s, e, n, b, d_csc_row, d_csc_ptr, flags + 1);
    GF_CHECK_LAUNCH("unpack_sorted csc");
    GF_CHECK_CUDA(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
    GF_CHECK_CUDA(cudaStreamSynchronize(s));
  } else {
    std::vector<int64_t> zeros(n + 1, 0);
    GF_CHECK_CUDA(cudaMemcpyAsync(d_row_ptr, zeros.data(), sizeof(int64_t) * (n + 1),
                                  cudaMemcpyHostToDevice, s));
    GF_CHECK_CUDA(cudaMemcpyAsync(d_csc_ptr, zeros.data(), sizeof(int64_t) * (n + 1),
                                  cudaMemcpyHostToDevice, s));
    GF_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  if (hflags[0] != ~0ull) {
    if (bad) *bad = static_cast<int64_t>(hflags[0]);
    set_error("from_coo: node id out of range for input edge " + std::to_string(hflags[0]));
    rc = GF_ERR_GRAPH;
  } else if (hflags[1] != ~0ull) {
    if (bad) *bad = -2 - static_cast<int64_t>(hflags[1]);
    set_error("from_coo: duplicate edge at sorted position " + std::to_string(hflags[1]));
    rc = GF_ERR_GRAPH;
  }
  cudaFreeAsync(k_ds, s);
  cudaFreeAsync(k_sd, s);
  cudaFreeAsync(k_ds_s, s);
  cudaFreeAsync(k_sd_s, s);
  cudaFreeAsync(flags, s);
  cudaStreamSynchronize(s);
  return rc;
}


extern "C" int gf_graph_set_split_len(gf_graph_t g, int64_t split_len, void* stream) {
  if (!g || split_len < 1) {
    gfb::set_error("gf_graph_set_split_len: null graph or split_len < 1");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  int rc = gfb::build_cta_table(g->row_sched, g->n_cta_rows, split_len, &g->row_cta,
                                g->row_cta_blocks, g->row_parts, s);
  if (!rc)
    rc = gfb::build_cta_table(g->col_sched, g->n_cta_cols, split_len, &g->col_cta,
                              g->col_cta_blocks, g->col_parts, s);
  return rc;
}

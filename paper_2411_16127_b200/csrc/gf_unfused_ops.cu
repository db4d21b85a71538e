// The reference's single-step operators (kernels.hpp:18-117 forward steps,
// autograd.hpp:33-170 backward steps) as device ops over multi-head E x H
// edge tensors in CSR order.  They are the building blocks of the unfused
// schedule — 3 forward launches, 5 backward launches (autograd.hpp:196-203)
// — which the fused path exists to beat; every one is its own kernel here so
// the unfused arm of the ablation moves the E x H intermediates through HBM
// exactly as the reference's counter model says it does.
//
//   sddmm            sddmm_edges (edge-parallel)                  kernels.hpp:18-47,106-117
//   edge_softmax     softmax_rows (warp per row, 3 sweeps)        kernels.hpp:65-82
//   spmm             fwd_fast/fwd_generic MODE 2 (CSR rows)       kernels.hpp:85-102
//   l2_normalize     l2_rows                                      kernels.hpp:50-61
//   spmm_backward    dP: sddmm_edges on (V[src], dO[dst]);        autograd.hpp:33-58
//                    dV: MODE 3 over the CSC view (P via perm)
//   softmax_backward softmax_bwd_rows                             autograd.hpp:62-73
//   l2 backward      l2_rows_bwd                                  autograd.hpp:76-95
//   sddmm_backward   dot: dK = MODE 2 rows, dQ = MODE 3 columns;  autograd.hpp:102-154
//                    add: add_grad (rows -> der, columns -> del)
// Owner-computes everywhere (no atomics): deterministic.
#include <algorithm>
#include <mutex>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

int grid_for(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 16, (work + 255) / 256)));
}

// CSC slot s of column u (destination v = csc_row[s]) -> CSR edge id: the
// position of u in row v's ascending source list (binary search).
__global__ void csc_perm_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                const int32_t* __restrict__ csc_ptr,
                                const int32_t* __restrict__ csc_row, int n,
                                int32_t* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (gridDim.x * blockDim.x) >> 5) {
    const int b = csc_ptr[u], e = csc_ptr[u + 1];
    for (int s = b + lane; s < e; s += 32) {
      const int v = csc_row[s];
      int lo = row_ptr[v], hi = row_ptr[v + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (col[mid] < u)
          lo = mid + 1;
        else
          hi = mid;
      }
      perm[s] = lo;
    }
  }
}

// softmax_backward per (row, head): t = sum_row P dP; dS = P (dP - t).
// Same contiguous-segment lane mapping as softmax_rows.
template <typename T>
__global__ void __launch_bounds__(256) softmax_bwd_rows(const int32_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ order, int n,
                                                        int H, const T* __restrict__ P,
                                                        const T* __restrict__ dP,
                                                        T* __restrict__ dS) {
  const int lane = threadIdx.x & 31;
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slot >= n) return;
  const int v = __ldg(order + slot);
  const size_t base = static_cast<size_t>(__ldg(ptr + v)) * H;
  const size_t len = static_cast<size_t>(__ldg(ptr + v + 1)) * H - base;
  if (32 % H == 0) {
    T t = T(0);
    for (size_t i = lane; i < len; i += 32) t += ld_edge(P + base + i) * ld_edge(dP + base + i);
    for (int o = H; o < 32; o <<= 1) t += __shfl_xor_sync(kFull, t, o);
    for (size_t i = lane; i < len; i += 32) {
      const T p = ld_edge(P + base + i);
      dS[base + i] = p * (ld_edge(dP + base + i) - t);
    }
  } else if (lane < H) {
    T t = T(0);
    for (size_t i = lane; i < len; i += H) t += ld_edge(P + base + i) * ld_edge(dP + base + i);
    for (size_t i = lane; i < len; i += H) {
      const T p = ld_edge(P + base + i);
      dS[base + i] = p * (ld_edge(dP + base + i) - t);
    }
  }
}

// Add-SDDMM backward (autograd.hpp:107-118), owner-computes per node and head:
//   COL = false: der[v,h] = sum over CSR row v   of dS[e,h] lrelu'(el[u,h] + er[v,h])
//   COL = true : del[u,h] = sum over CSC column u of dS[perm[s],h] lrelu'(...)
template <typename T, bool COL>
__global__ void __launch_bounds__(256) add_grad(const int32_t* __restrict__ ptr,
                                                const int32_t* __restrict__ idx,
                                                const int32_t* __restrict__ perm,
                                                const int32_t* __restrict__ order, int n, int H,
                                                T slope, const T* __restrict__ el,
                                                const T* __restrict__ er,
                                                const T* __restrict__ dS, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slot >= n) return;
  const int r = __ldg(order + slot);
  const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
  auto term = [&](int s, int h) {
    const int o = __ldg(idx + s);  // the other endpoint
    const int ei = COL ? __ldg(perm + s) : s;
    const T pre = COL ? __ldg(el + static_cast<size_t>(r) * H + h) + __ldg(er + static_cast<size_t>(o) * H + h)
                      : __ldg(el + static_cast<size_t>(o) * H + h) + __ldg(er + static_cast<size_t>(r) * H + h);
    return ld_edge(dS + static_cast<size_t>(ei) * H + h) * lrelu_grad(pre, slope);
  };
  if (32 % H == 0) {
    const int h = lane % H, step = 32 / H;
    T acc = T(0);
    for (int s = b + lane / H; s < e; s += step) acc += term(s, h);
    for (int o = H; o < 32; o <<= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane < H) out[static_cast<size_t>(r) * H + h] = acc;
  } else if (lane < H) {
    T acc = T(0);
    for (int s = b; s < e; ++s) acc += term(s, lane);
    out[static_cast<size_t>(r) * H + lane] = acc;
  }
}

// Per-head row L2 normalisation y = x / max(||x||, eps) (kernels.hpp:50-61)
// and its backward (autograd.hpp:76-95); one warp per (node, head) row with
// lanes over the D features (coalesced), sums by warp shuffles.
template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

template <typename T>
__global__ void __launch_bounds__(256) l2_rows(int64_t rows, int D, const T* __restrict__ X,
                                               T* __restrict__ Y, T eps) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const T* x = X + r * D;
    T sq = T(0);
    for (int c = lane; c < D; c += 32) sq += x[c] * x[c];
    const T nrm = sqrt(warp_sum(sq));
    const T den = nrm < eps ? eps : nrm;
    for (int c = lane; c < D; c += 32) Y[r * D + c] = x[c] / den;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) l2_rows_bwd(int64_t rows, int D, const T* __restrict__ X,
                                                   const T* __restrict__ dY, T* __restrict__ dX,
                                                   T eps) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const T* x = X + r * D;
    const T* dy = dY + r * D;
    T sq = T(0);
    for (int c = lane; c < D; c += 32) sq += x[c] * x[c];
    const T nrm = sqrt(warp_sum(sq));
    if (nrm <= eps) {
      for (int c = lane; c < D; c += 32) dX[r * D + c] = dy[c] / eps;
      continue;
    }
    T dot = T(0);
    for (int c = lane; c < D; c += 32) dot += x[c] / nrm * dy[c];
    dot = warp_sum(dot);
    for (int c = lane; c < D; c += 32) dX[r * D + c] = (dy[c] - x[c] / nrm * dot) / nrm;
  }
}

template <typename T>
FwdArgs<T> base_args(const DevGraph& g, int H, int D, bool csc) {
  FwdArgs<T> a{};
  a.ptr = csc ? g.csc_ptr : g.row_ptr;
  a.idx = csc ? g.csc_row : g.col;
  a.order = csc ? g.col_order : g.row_order;
  a.sched = csc ? g.col_sched : g.row_sched;
  a.n_small = csc ? g.n_small_cols : g.n_small_rows;
  a.n_empty = csc ? g.n_empty_cols : g.n_empty_rows;
  a.e = csc ? g.e_csc : g.e;
  a.n = csc ? g.active_cols() : g.active_rows();
  a.n_cta = csc ? g.n_cta_cols : g.n_cta_rows;
  a.cta_tab = csc ? g.col_cta : g.row_cta;
  a.cta_blocks = csc ? g.col_cta_blocks : g.row_cta_blocks;
  a.parts = csc ? g.col_parts : g.row_parts;
  a.H = H;
  a.D = D;
  a.F = H * D;
  a.LPH = 1;
  a.scale = T(1);
  a.slope = T(0.2);
  return a;
}

// out[r] = scale * sum_{slot in r} w(slot) * X[idx[slot]] over the CSR rows
// (csc = false, w = ES[slot]) or the CSC columns (csc = true, w = ES[perm[slot]]).
template <typename T>
int spmm_pass(DevGraph& g, int H, int D, bool csc, const T* w, const T* X, T* out, T scale,
              cudaStream_t s) {
  FwdArgs<T> a = base_args<T>(g, H, D, csc);
  a.ES = w;
  a.V = X;
  a.O = out;
  a.scale = scale;
  if (csc) {
    if (int rc = ensure_csc_perm(g, s)) return rc;
    a.eperm = g.csc_perm;
  }
  return launch_fwd_mode<T>(g, a, GF_ADD, csc ? 3 : 2, s);
}

bool whole_graph(const DevGraph& g, const char* who) {
  if (g.skip_empty || g.e_csc != g.e) {
    set_error(std::string(who) + ": needs an unsharded graph (CSR and CSC over the same edges)");
    return false;
  }
  return true;
}

template <typename T>
int l2_launch(int64_t n, int H, int D, const T* X, T* Y, cudaStream_t s, T eps = T(1e-12)) {
  if (n == 0) return GF_OK;
  l2_rows<T><<<grid_for(n * H * 32), 256, 0, s>>>(n * H, D, X, Y, eps);
  GF_CHECK_LAUNCH("l2_rows");
  return GF_OK;
}

template <typename T>
int l2_bwd_launch(int64_t n, int H, int D, const T* X, const T* dY, T* dX, cudaStream_t s,
                  T eps = T(1e-12)) {
  if (n == 0) return GF_OK;
  l2_rows_bwd<T><<<grid_for(n * H * 32), 256, 0, s>>>(n * H, D, X, dY, dX, eps);
  GF_CHECK_LAUNCH("l2_rows_bwd");
  return GF_OK;
}

template <typename T>
int sddmm_backward_impl(DevGraph& g, const gf_attn_desc& d, const T* Q, const T* K, const T* dS,
                        T* dQ, T* dK, cudaStream_t s) {
  const int H = d.heads, D = d.head_dim;
  if (d.variant == GF_ADD) {
    if (int rc = ensure_csc_perm(g, s)) return rc;
    const int rows = g.active_rows(), cols = g.active_cols();
    if (rows > 0) {
      add_grad<T, false><<<static_cast<int>((int64_t(rows) * 32 + 255) / 256), 256, 0, s>>>(
          g.row_ptr, g.col, nullptr, g.row_order, rows, H, static_cast<T>(d.slope), Q, K, dS, dK);
      GF_CHECK_LAUNCH("add_grad rows");
    }
    if (cols > 0) {
      add_grad<T, true><<<static_cast<int>((int64_t(cols) * 32 + 255) / 256), 256, 0, s>>>(
          g.csc_ptr, g.csc_row, g.csc_perm, g.col_order, cols, H, static_cast<T>(d.slope), Q, K,
          dS, dQ);
      GF_CHECK_LAUNCH("add_grad cols");
    }
    return GF_OK;
  }
  const T scale = static_cast<T>(d.scale);
  const size_t nf = static_cast<size_t>(g.n) * H * D;
  if (!d.l2) {  // dK over in-edges (CSR rows, gather Q[src]); dQ over out-edges (CSC, K[dst])
    if (int rc = spmm_pass<T>(g, H, D, false, dS, Q, dK, scale, s)) return rc;
    return spmm_pass<T>(g, H, D, true, dS, K, dQ, scale, s);
  }
  // AGNN: gradients w.r.t. the normalised rows, then through the normalisation
  T* tmp = nullptr;
  GF_CHECK_CUDA(gfb::scratch_alloc(&tmp, sizeof(T) * nf * 4, s));
  T *qn = tmp, *kn = tmp + nf, *gq = tmp + 2 * nf, *gk = tmp + 3 * nf;
  int rc = l2_launch<T>(g.n, H, D, Q, qn, s);
  if (!rc) rc = l2_launch<T>(g.n, H, D, K, kn, s);
  if (!rc) rc = spmm_pass<T>(g, H, D, false, dS, qn, gk, scale, s);
  if (!rc) rc = spmm_pass<T>(g, H, D, true, dS, kn, gq, scale, s);
  if (!rc) rc = l2_bwd_launch<T>(g.n, H, D, Q, gq, dQ, s);
  if (!rc) rc = l2_bwd_launch<T>(g.n, H, D, K, gk, dK, s);
  cudaFreeAsync(tmp, s);
  return rc;
}

int check_desc(const gf_attn_desc* d, const char* who) {
  if (!d || (d->dtype != GF_F32 && d->dtype != GF_F64) ||
      (d->variant != GF_DOT && d->variant != GF_ADD) || d->heads < 1 || d->head_dim < 1 ||
      (d->variant == GF_ADD && d->l2) || d->reserved != 0) {
    set_error(std::string(who) + ": invalid descriptor (the single-step ops take explicit "
              "el / er: no descriptor flags)");
    return GF_ERR_INVALID;
  }
  return GF_OK;
}

bool bad_shape(gf_graph_t g, int32_t dtype, int32_t heads, int32_t head_dim, const char* who) {
  if (!g || (dtype != GF_F32 && dtype != GF_F64) || heads < 1 || head_dim < 1) {
    set_error(std::string(who) + ": invalid arguments");
    return true;
  }
  return false;
}

}  // namespace

int ensure_csc_perm(DevGraph& g, cudaStream_t s) {
  static std::mutex mu;  // graphs are shareable across host threads
  std::lock_guard<std::mutex> lock(mu);
  if (g.csc_perm || g.e == 0) return GF_OK;
  if (!whole_graph(g, "csc_perm")) return GF_ERR_UNSUPPORTED;
  GF_CHECK_CUDA(cudaMalloc(&g.csc_perm, sizeof(int32_t) * g.e));
  const int blocks = static_cast<int>(std::min<int64_t>(148 * 32, (int64_t(g.n) * 32 + 255) / 256 + 1));
  csc_perm_kernel<<<blocks, 256, 0, s>>>(g.row_ptr, g.col, g.csc_ptr, g.csc_row, g.n, g.csc_perm);
  GF_CHECK_LAUNCH("csc_perm_kernel");
  return GF_OK;
}

}  // namespace gfb

using gfb::DevGraph;

// ---------------------------------------------------------------- C-ABI --
extern "C" int gf_sddmm(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                        void* S, void* stream) {
  if (int rc = gfb::check_desc(desc, "gf_sddmm")) return rc;
  if (!g) return gfb::set_error("gf_sddmm: null graph"), GF_ERR_INVALID;
  auto s = static_cast<cudaStream_t>(stream);
  if (desc->dtype == GF_F32) {
    auto a = gfb::base_args<float>(*g, desc->heads, desc->head_dim, false);
    a.Q = static_cast<const float*>(Q), a.K = static_cast<const float*>(K);
    a.scale = static_cast<float>(desc->scale), a.slope = static_cast<float>(desc->slope);
    a.l2 = desc->l2;
    return gfb::launch_sddmm_edges<float>(*g, a, desc->variant, static_cast<float*>(S), s);
  }
  auto a = gfb::base_args<double>(*g, desc->heads, desc->head_dim, false);
  a.Q = static_cast<const double*>(Q), a.K = static_cast<const double*>(K);
  a.scale = desc->scale, a.slope = desc->slope;
  a.l2 = desc->l2;
  return gfb::launch_sddmm_edges<double>(*g, a, desc->variant, static_cast<double*>(S), s);
}

extern "C" int gf_edge_softmax(gf_graph_t g, int32_t dtype, int32_t heads, const void* S, void* P,
                               void* stream) {
  if (gfb::bad_shape(g, dtype, heads, 1, "gf_edge_softmax")) return GF_ERR_INVALID;
  auto s = static_cast<cudaStream_t>(stream);
  if (dtype == GF_F32) {
    auto a = gfb::base_args<float>(*g, heads, 1, false);
    return gfb::launch_softmax_rows<float>(*g, a, GF_ADD, static_cast<const float*>(S),
                                           static_cast<float*>(P), s);
  }
  auto a = gfb::base_args<double>(*g, heads, 1, false);
  return gfb::launch_softmax_rows<double>(*g, a, GF_ADD, static_cast<const double*>(S),
                                          static_cast<double*>(P), s);
}

extern "C" int gf_spmm(gf_graph_t g, int32_t dtype, int32_t heads, int32_t head_dim,
                       const void* P, const void* V, void* O, void* stream) {
  if (gfb::bad_shape(g, dtype, heads, head_dim, "gf_spmm")) return GF_ERR_INVALID;
  auto s = static_cast<cudaStream_t>(stream);
  return dtype == GF_F32
             ? gfb::spmm_pass<float>(*g, heads, head_dim, false, static_cast<const float*>(P),
                                     static_cast<const float*>(V), static_cast<float*>(O), 1.f, s)
             : gfb::spmm_pass<double>(*g, heads, head_dim, false, static_cast<const double*>(P),
                                      static_cast<const double*>(V), static_cast<double*>(O), 1.0,
                                      s);
}

extern "C" int gf_l2_normalize_rows(int32_t dtype, int64_t n, int32_t heads, int32_t head_dim,
                                    const void* X, void* Y, double eps, void* stream) {
  if (n < 0 || heads < 1 || head_dim < 1 || (dtype != GF_F32 && dtype != GF_F64) || !(eps > 0))
    return gfb::set_error("gf_l2_normalize_rows: invalid arguments (eps must be > 0)"),
           GF_ERR_INVALID;
  auto s = static_cast<cudaStream_t>(stream);
  return dtype == GF_F32 ? gfb::l2_launch<float>(n, heads, head_dim, static_cast<const float*>(X),
                                                 static_cast<float*>(Y), s, static_cast<float>(eps))
                         : gfb::l2_launch<double>(n, heads, head_dim, static_cast<const double*>(X),
                                                  static_cast<double*>(Y), s, eps);
}

extern "C" int gf_l2_normalize_backward(int32_t dtype, int64_t n, int32_t heads, int32_t head_dim,
                                        const void* X, const void* dY, void* dX, double eps,
                                        void* stream) {
  if (n < 0 || heads < 1 || head_dim < 1 || (dtype != GF_F32 && dtype != GF_F64) || !(eps > 0))
    return gfb::set_error("gf_l2_normalize_backward: invalid arguments (eps must be > 0)"),
           GF_ERR_INVALID;
  auto s = static_cast<cudaStream_t>(stream);
  return dtype == GF_F32
             ? gfb::l2_bwd_launch<float>(n, heads, head_dim, static_cast<const float*>(X),
                                         static_cast<const float*>(dY), static_cast<float*>(dX), s,
                                         static_cast<float>(eps))
             : gfb::l2_bwd_launch<double>(n, heads, head_dim, static_cast<const double*>(X),
                                          static_cast<const double*>(dY), static_cast<double*>(dX),
                                          s, eps);
}

extern "C" int gf_spmm_backward(gf_graph_t g, int32_t dtype, int32_t heads, int32_t head_dim,
                                const void* P, const void* V, const void* dO, void* dP, void* dV,
                                void* stream) {
  if (gfb::bad_shape(g, dtype, heads, head_dim, "gf_spmm_backward")) return GF_ERR_INVALID;
  if (!gfb::whole_graph(*g, "gf_spmm_backward")) return GF_ERR_UNSUPPORTED;
  auto s = static_cast<cudaStream_t>(stream);
  // dP[e,h] = <dO[dst], V[src]>: the dot SDDMM with Q := V (source), K := dO (destination)
  gf_attn_desc d{dtype, GF_DOT, 0, heads, head_dim, 0, 1.0, 0.0};
  if (int rc = gf_sddmm(g, &d, V, dO, dP, stream)) return rc;
  return dtype == GF_F32
             ? gfb::spmm_pass<float>(*g, heads, head_dim, true, static_cast<const float*>(P),
                                     static_cast<const float*>(dO), static_cast<float*>(dV), 1.f, s)
             : gfb::spmm_pass<double>(*g, heads, head_dim, true, static_cast<const double*>(P),
                                      static_cast<const double*>(dO), static_cast<double*>(dV),
                                      1.0, s);
}

extern "C" int gf_softmax_backward(gf_graph_t g, int32_t dtype, int32_t heads, const void* P,
                                   const void* dP, void* dS, void* stream) {
  if (gfb::bad_shape(g, dtype, heads, 1, "gf_softmax_backward")) return GF_ERR_INVALID;
  if (heads > 32) return gfb::set_error("gf_softmax_backward: heads <= 32"), GF_ERR_UNSUPPORTED;
  const int n = g->active_rows();
  if (n == 0) return GF_OK;
  auto s = static_cast<cudaStream_t>(stream);
  const int blocks = static_cast<int>((static_cast<int64_t>(n) * 32 + 255) / 256);
  if (dtype == GF_F32)
    gfb::softmax_bwd_rows<float><<<blocks, 256, 0, s>>>(
        g->row_ptr, g->row_order, n, heads, static_cast<const float*>(P),
        static_cast<const float*>(dP), static_cast<float*>(dS));
  else
    gfb::softmax_bwd_rows<double><<<blocks, 256, 0, s>>>(
        g->row_ptr, g->row_order, n, heads, static_cast<const double*>(P),
        static_cast<const double*>(dP), static_cast<double*>(dS));
  GF_CHECK_LAUNCH("softmax_bwd_rows");
  return GF_OK;
}

extern "C" int gf_sddmm_backward(gf_graph_t g, const gf_attn_desc* desc, const void* Q,
                                 const void* K, const void* dS, void* dQ, void* dK, void* stream) {
  if (int rc = gfb::check_desc(desc, "gf_sddmm_backward")) return rc;
  if (!g) return gfb::set_error("gf_sddmm_backward: null graph"), GF_ERR_INVALID;
  if (!gfb::whole_graph(*g, "gf_sddmm_backward")) return GF_ERR_UNSUPPORTED;
  if (desc->heads > 32) return gfb::set_error("gf_sddmm_backward: heads <= 32"), GF_ERR_UNSUPPORTED;
  auto s = static_cast<cudaStream_t>(stream);
  return desc->dtype == GF_F32
             ? gfb::sddmm_backward_impl<float>(*g, *desc, static_cast<const float*>(Q),
                                               static_cast<const float*>(K),
                                               static_cast<const float*>(dS),
                                               static_cast<float*>(dQ), static_cast<float*>(dK), s)
             : gfb::sddmm_backward_impl<double>(*g, *desc, static_cast<const double*>(Q),
                                                static_cast<const double*>(K),
                                                static_cast<const double*>(dS),
                                                static_cast<double*>(dQ), static_cast<double*>(dK),
                                                s);
}

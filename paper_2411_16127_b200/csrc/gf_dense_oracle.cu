// dense_oracle_forward (kernels.hpp:122-166) on the device: the reference's
// own masked dense test oracle, part of its public kernels.hpp API (its unit
// tests and acceptance criterion 1 call it).  It materialises the N x N score
// matrix S[v][u] of edge u -> v, applies a row softmax over the mask support
// in ascending u, and multiplies densely, in the reference's arithmetic order:
//   1. zero S, O and the mask (n <= 4096: at most 16 M entries);
//   2. one thread per edge writes its score (dot over L2-normalised rows when
//      desc->l2, add + LeakyReLU otherwise) and sets mask[v][u];
//   3. one thread per row v scans u = 0..n-1: zmax, zsum, then
//      O[v,:] += p * V[u,:] for each masked u (empty rows stay zero).
// Deliberately dense and O(N^2): it is the independent check of the sparse
// path, not a fast path.
#include <math_constants.h>

#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

template <typename T>
__device__ T row_norm(const T* __restrict__ x, int64_t cols) {
  T sq = 0;
  for (int64_t c = 0; c < cols; ++c) sq = sq + x[c] * x[c];
  return sqrt(sq);
}

template <typename T>
__global__ void dense_scores(int64_t n, int64_t e, const int64_t* __restrict__ src,
                             const int64_t* __restrict__ dst, int32_t variant, int32_t l2,
                             int64_t qk_cols, double scale, double slope,
                             const T* __restrict__ Q, const T* __restrict__ K, T* __restrict__ S,
                             unsigned char* __restrict__ mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t u = src[i], v = dst[i];
    mask[v * n + u] = 1;
    T s;
    if (variant == GF_DOT) {
      const T* q = Q + u * qk_cols;
      const T* k = K + v * qk_cols;
      T nq = 1, nk = 1;
      if (l2) {  // l2_normalize_rows(., 1e-12): x / max(||x||, eps)
        nq = max(row_norm(q, qk_cols), T(1e-12));
        nk = max(row_norm(k, qk_cols), T(1e-12));
      }
      T acc = 0;
      for (int64_t c = 0; c < qk_cols; ++c) {
        const T a = l2 ? q[c] / nq : q[c];
        const T b = l2 ? k[c] / nk : k[c];
        acc = acc + a * b;
      }
      s = static_cast<T>(scale) * acc;
    } else {
      const T x = Q[u] + K[v];
      s = x >= T(0) ? x : static_cast<T>(slope) * x;
    }
    S[v * n + u] = s;
  }
}

template <typename T>
__global__ void dense_softmax_product(int64_t n, int64_t v_cols, const T* __restrict__ S,
                                      const unsigned char* __restrict__ mask,
                                      const T* __restrict__ V, T* __restrict__ O) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= n) return;
  const T* srow = S + v * n;
  const unsigned char* mrow = mask + v * n;
  T zmax = -CUDART_INF;
  for (int64_t u = 0; u < n; ++u)
    if (mrow[u]) zmax = max(zmax, srow[u]);
  if (zmax == T(-CUDART_INF)) return;  // empty row
  T zsum = 0;
  for (int64_t u = 0; u < n; ++u)
    if (mrow[u]) zsum = zsum + exp(srow[u] - zmax);
  T* o = O + v * v_cols;
  for (int64_t u = 0; u < n; ++u) {
    if (!mrow[u]) continue;
    const T p = exp(srow[u] - zmax) / zsum;
    for (int64_t c = 0; c < v_cols; ++c) o[c] = o[c] + p * V[u * v_cols + c];
  }
}

template <typename T>
int dense_oracle_impl(int64_t n, int64_t e, const int64_t* src, const int64_t* dst,
                      const gf_attn_desc& d, int64_t v_cols, const T* Q, const T* K, const T* V,
                      T* S, T* O, cudaStream_t s) {
  unsigned char* mask = nullptr;
  GF_CHECK_CUDA(scratch_alloc(&mask, static_cast<size_t>(n) * n, s));
  GF_CHECK_CUDA(cudaMemsetAsync(mask, 0, static_cast<size_t>(n) * n, s));
  GF_CHECK_CUDA(cudaMemsetAsync(S, 0, sizeof(T) * n * n, s));
  GF_CHECK_CUDA(cudaMemsetAsync(O, 0, sizeof(T) * n * v_cols, s));
  int rc = GF_OK;
  if (e > 0) {
    const int blocks = static_cast<int>(std::min<int64_t>((e + 255) / 256, 148 * 16));
    dense_scores<T><<<blocks, 256, 0, s>>>(n, e, src, dst, d.variant, d.l2, d.head_dim, d.scale,
                                           d.slope, Q, K, S, mask);
    if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
    if (!rc) {
      dense_softmax_product<T><<<static_cast<int>((n + 127) / 128), 128, 0, s>>>(n, v_cols, S, mask,
                                                                                V, O);
      if (cudaGetLastError() != cudaSuccess) rc = GF_ERR_CUDA;
    }
    if (rc) set_error("gf_dense_oracle_forward: launch failed");
  }
  cudaFreeAsync(mask, s);
  return rc;
}

}  // namespace
}  // namespace gfb

extern "C" int gf_dense_oracle_forward(int64_t n, int64_t e, const int64_t* coo_src,
                                       const int64_t* coo_dst, const gf_attn_desc* desc,
                                       int64_t v_cols, const void* Q, const void* K,
                                       const void* V, void* S, void* O, void* stream) {
  if (!desc || n < 0 || e < 0 || v_cols < 0 || (desc->dtype != GF_F32 && desc->dtype != GF_F64) ||
      (desc->variant != GF_DOT && desc->variant != GF_ADD) || desc->head_dim < 1) {
    gfb::set_error("gf_dense_oracle_forward: invalid descriptor or sizes");
    return GF_ERR_INVALID;
  }
  if (n > 4096) {
    gfb::set_error("dense_oracle_forward: N > 4096");
    return GF_ERR_INVALID;
  }
  if (n == 0) return GF_OK;
  if ((e > 0 && (!coo_src || !coo_dst || !Q || !K)) || !S || (v_cols > 0 && (!V || !O))) {
    gfb::set_error("gf_dense_oracle_forward: null operand");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  return desc->dtype == GF_F32
             ? gfb::dense_oracle_impl<float>(n, e, coo_src, coo_dst, *desc, v_cols,
                                             static_cast<const float*>(Q),
                                             static_cast<const float*>(K),
                                             static_cast<const float*>(V), static_cast<float*>(S),
                                             static_cast<float*>(O), s)
             : gfb::dense_oracle_impl<double>(n, e, coo_src, coo_dst, *desc, v_cols,
                                              static_cast<const double*>(Q),
                                              static_cast<const double*>(K),
                                              static_cast<const double*>(V),
                                              static_cast<double*>(S), static_cast<double*>(O), s);
}

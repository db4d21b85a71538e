// Merge of source-phased forward partials (multi-GPU overlap, SURVEY §8(e)
// "chunked all-gather overlapped with compute on locally-sourced edges
// first").  A row-sharded rank can start its forward on the edges whose
// sources it owns while the other ranks' source rows are still arriving: the
// forward runs once per source block k over the sub-graph of its rows'
// in-edges from block k (rows stay sorted by source, so each is a contiguous
// slice of the row), writing a normalised partial O_k and record {m_k,
// log2 l_k, aux}.  This kernel combines the parts per (row, head):
//   m = max_k m_k,  w_k = l_k e^(m_k - m),  L = sum_k w_k,
//   O = sum_k w_k O_k / L,  record = {m, log2 L, aux, delta (untouched)}
// which is the softmax over the union of the edge sets (the parts are
// disjoint).  Parts whose sub-graph row is empty are skipped (their O_k /
// record slots were never written); rows empty in every part are left
// untouched, like the un-phased sharded forward (skip-empty graphs).
#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

constexpr int kMaxParts = 8;

template <typename T>
struct Parts {
  const int32_t* rp[kMaxParts];  // row pointer of each part's sub-graph (row-relative)
  const T* O[kMaxParts];         // rows x F
  const T* rec[kMaxParts];       // rows x H x 4
  int n;
};

// One warp per row: lanes own heads for the weights, then features.
template <typename T>
__global__ void __launch_bounds__(256) merge_parts(const Parts<T> p, int64_t rows, int H, int D,
                                                   T* __restrict__ O, T* __restrict__ rec) {
  __shared__ T wsh[8][kMaxParts][32];
  __shared__ T lsh[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int F = H * D;
  for (int64_t v = blockIdx.x * 8LL + warp; v < rows; v += gridDim.x * 8LL) {
    unsigned live = 0;  // parts with edges in this row
    for (int k = 0; k < p.n; ++k)
      if (__ldg(p.rp[k] + v + 1) > __ldg(p.rp[k] + v)) live |= 1u << k;
    if (!live) continue;  // warp-uniform
    for (int h = lane; h < H && h < 32; h += 32) {
      T m = ninf<T>(), aux = T(0);
      for (int k = 0; k < p.n; ++k)
        if (live >> k & 1) {
          const T* r = p.rec[k] + 4 * (v * H + h);
          m = max(m, r[0]);
          aux = r[2];
        }
      T L = T(0);
      for (int k = 0; k < p.n; ++k) {
        T w = T(0);
        if (live >> k & 1) {
          const T* r = p.rec[k] + 4 * (v * H + h);
          w = r[0] == ninf<T>() ? T(0) : ex2((r[0] - m) * l2e<T>() + r[1]);
        }
        wsh[warp][k][h] = w;
        L += w;
      }
      lsh[warp][h] = L;
      T* out = rec + 4 * (v * H + h);
      out[0] = L == T(0) ? ninf<T>() : m;
      out[1] = L == T(0) ? T(0) : lg2(L);
      out[2] = aux;
    }
    __syncwarp();
    for (int f = lane; f < F; f += 32) {
      const int h = f / D;
      const T L = lsh[warp][h];
      T o = T(0);
      for (int k = 0; k < p.n; ++k)
        if (live >> k & 1) o += wsh[warp][k][h] * __ldg(p.O[k] + v * F + f);
      O[v * F + f] = L == T(0) ? T(0) : o / L;
    }
    __syncwarp();
  }
}

template <typename T>
int merge_launch(int64_t rows, int H, int D, int n, const int32_t* const* rp,
                 const void* const* Op, const void* const* recp, void* O, void* rec,
                 cudaStream_t s) {
  Parts<T> p;
  p.n = n;
  for (int k = 0; k < n; ++k) {
    p.rp[k] = rp[k];
    p.O[k] = static_cast<const T*>(Op[k]);
    p.rec[k] = static_cast<const T*>(recp[k]);
  }
  const int blocks = static_cast<int>(std::min<int64_t>(148 * 16, (rows + 7) / 8));
  merge_parts<T><<<blocks, 256, 0, s>>>(p, rows, H, D, static_cast<T*>(O), static_cast<T*>(rec));
  GF_CHECK_LAUNCH("merge_parts");
  return GF_OK;
}

}  // namespace
}  // namespace gfb

extern "C" int gf_attn_merge_parts(int32_t dtype, int64_t rows, int32_t heads, int32_t head_dim,
                                   int32_t parts, const int32_t* const* row_ptrs,
                                   const void* const* O_parts, const void* const* rec_parts,
                                   void* O, void* rec, void* stream) {
  if (rows < 0 || heads < 1 || heads > 32 || head_dim < 1 || parts < 1 ||
      parts > gfb::kMaxParts || !row_ptrs || !O_parts || !rec_parts || !O || !rec ||
      (dtype != GF_F32 && dtype != GF_F64)) {
    gfb::set_error("gf_attn_merge_parts: invalid arguments (1 <= parts <= 8, heads <= 32)");
    return GF_ERR_INVALID;
  }
  for (int k = 0; k < parts; ++k)
    if (!row_ptrs[k] || !O_parts[k] || !rec_parts[k]) {
      gfb::set_error("gf_attn_merge_parts: null part");
      return GF_ERR_INVALID;
    }
  if (rows == 0) return GF_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dtype == GF_F32 ? gfb::merge_launch<float>(rows, heads, head_dim, parts, row_ptrs,
                                                    O_parts, rec_parts, O, rec, s)
                         : gfb::merge_launch<double>(rows, heads, head_dim, parts, row_ptrs,
                                                     O_parts, rec_parts, O, rec, s);
}

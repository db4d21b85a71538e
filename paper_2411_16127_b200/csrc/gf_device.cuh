// Device helpers shared by the fused attention kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gfb {

constexpr unsigned kFull = 0xffffffffu;

// 16-byte chunk of T: 4 floats or 2 doubles.
template <typename T>
struct Chunk {
  static constexpr int W = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void ld_chunk(const T* __restrict__ p, T (&x)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
  } else {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = v.x, x[1] = v.y;
  }
}

template <typename T>
__device__ __forceinline__ void st_chunk(T* __restrict__ p, const T (&x)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
  }
}

// exp(x): one MUFU.EX2 plus a multiply for fp32, full precision for fp64.
__device__ __forceinline__ float gexp(float x) { return exp2f(x * 1.4426950408889634f); }
__device__ __forceinline__ double gexp(double x) { return exp(x); }
__device__ __forceinline__ float glog(float x) { return logf(x); }
__device__ __forceinline__ double glog(double x) { return log(x); }

template <typename T>
__device__ __forceinline__ T ninf() {
  return -INFINITY;
}

// Softmax statistics per (row, head): (m, log l) with m the row max and l the
// sum of exp(s - m).  p = exp((s - m) - log l) keeps full relative precision
// for any score magnitude (a single fused lse = m + log l would lose
// ulp(|m|) absolute, i.e. ~6e-5 relative at |s| ~ 1e3 in fp32).
template <typename T>
__device__ __forceinline__ void ld_stat(const T* __restrict__ st, size_t i, T& m, T& ll) {
  if constexpr (sizeof(T) == 4) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(st) + i);
    m = v.x, ll = v.y;
  } else {
    const double2 v = __ldg(reinterpret_cast<const double2*>(st) + i);
    m = v.x, ll = v.y;
  }
}
template <typename T>
__device__ __forceinline__ void st_stat(T* st, size_t i, T m, T ll) {
  st[2 * i] = m;
  st[2 * i + 1] = ll;
}
template <typename T>
__device__ __forceinline__ T prob(T s, T m, T ll) {
  return gexp((s - m) - ll);
}

template <typename T>
__device__ __forceinline__ T lrelu(T x, T slope) {
  return x >= T(0) ? x : slope * x;  // kernels.hpp:44
}
template <typename T>
__device__ __forceinline__ T lrelu_grad(T pre, T slope) {
  return pre > T(0) ? T(1) : slope;  // autograd.hpp:113 (kink takes the slope)
}

// Sum of per-chunk partials over one head.  Lanes of an edge group (LPE
// lanes, aligned) hold chunk c + k*LPE for k < CPL; a head spans GD
// consecutive chunks (GD a power of two).  After the call every lane holds
// its head's total in x[k].
template <int LPE, int CPL, typename T>
__device__ __forceinline__ void head_sum(T (&x)[CPL], int gd) {
  const int lim = gd < LPE ? gd : LPE;
#pragma unroll
  for (int off = 1; off < LPE; off <<= 1) {
    if (off < lim) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[k] += __shfl_xor_sync(kFull, x[k], off);
    }
  }
  if constexpr (CPL > 1) {
    if (gd > LPE) {
      const int gk = gd / LPE;  // consecutive k per head
      T t[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int k0 = (k / gk) * gk;
        T s = T(0);
#pragma unroll
        for (int j = 0; j < CPL; ++j)
          if (j >= k0 && j < k0 + gk) s += x[j];
        t[k] = s;
      }
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[k] = t[k];
    }
  }
}

template <typename T>
__device__ __forceinline__ T inv_norm(T sq) {
  const T eps = T(1e-12);
  const T nrm = sqrt(sq);
  return T(1) / (nrm < eps ? eps : nrm);  // 1 / max(||x||, eps), kernels.hpp:57
}

// ------------------------------------------------ generic (any-shape) path --
// Lane h < H owns head h; scores are computed serially over D.  Works on any
// argument struct with Q, K, F, D, H, l2, scale, slope (FwdArgs / BwdArgs).
constexpr int kGenericWarps = 4;

// Score of edge u -> v for head h.  kvs: K[v] staged in shared memory (or
// null to read global).  erh: er[v,h] (add).  rkh: 1/max(||K[v,h]||,eps)
// (AGNN).  rq_out: 1/max(||Q[u,h]||,eps) (AGNN).  pre_out: el+er (add).
template <typename T, int VAR, class A>
__device__ __forceinline__ T generic_score(const A& a, int u, int v, int h, const T* kvs, T erh,
                                           T rkh, T* rq_out = nullptr, T* pre_out = nullptr) {
  if constexpr (VAR == 0) {
    const T* q = a.Q + static_cast<size_t>(u) * a.F + h * a.D;
    const T* k = kvs ? kvs + h * a.D : a.K + static_cast<size_t>(v) * a.F + h * a.D;
    T d = T(0), qq = T(0);
    for (int j = 0; j < a.D; ++j) {
      const T x = __ldg(q + j);
      d += x * k[j];
      qq += x * x;
    }
    if (!a.l2) return a.scale * d;
    const T rq = inv_norm(qq);
    if (rq_out) *rq_out = rq;
    return a.scale * d * (rq * rkh);
  } else {
    const T pre = __ldg(a.Q + static_cast<size_t>(u) * a.H + h) + erh;
    if (pre_out) *pre_out = pre;
    return lrelu(pre, a.slope);
  }
}

// Per-row destination operands for lane h: er[v,h] (add) or the AGNN inverse
// norm of K[v,h] (dot + l2).
template <typename T, int VAR, class A>
__device__ __forceinline__ void generic_row_setup(const A& a, int v, int lane, const T* kvs,
                                                  T& erh, T& rkh) {
  erh = T(0);
  rkh = T(1);
  if (lane < a.H) {
    if constexpr (VAR == 1) {
      erh = __ldg(a.K + static_cast<size_t>(v) * a.H + lane);
    } else if (a.l2) {
      const T* k = kvs ? kvs + lane * a.D : a.K + static_cast<size_t>(v) * a.F + lane * a.D;
      T s = T(0);
      for (int j = 0; j < a.D; ++j) s += k[j] * k[j];
      rkh = inv_norm(s);
    }
  }
}

// Balanced split of [b, e) into `parts` contiguous slices (first `rem` get +1),
// the same rule the reference uses for warp_balance (schedule.cpp:42-60).
__device__ __forceinline__ void split_range(int b, int e, int parts, int i, int& sb, int& se) {
  const int len = e - b, base = len / parts, rem = len % parts;
  sb = b + i * base + (i < rem ? i : rem);
  se = sb + base + (i < rem ? 1 : 0);
}

}  // namespace gfb

// Device helpers shared by the fused attention kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gf_policy.h"

namespace gfb {

constexpr unsigned kFull = 0xffffffffu;
// Every thread of the grid prefetches its share of up to three node tables
// into L2 (prefetch.global.L2, one 128 B line per request).  A hint only:
// it never changes results, so it may run before pdl_wait.
__device__ __forceinline__ void l2_prefetch_tables(const void* const (&p)[3],
                                                   const int64_t (&len)[3]) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const char* b = static_cast<const char*>(p[k]);
    for (int64_t off = tid * 128; off < len[k]; off += nth * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(b + off));
  }
}

// PDL (gf_internal.cuh launch_k): wait for the previous grid's completion and
// memory before touching global memory; let the next grid be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

// Element-pair arithmetic: on sm_100 fp32 pairs map to FFMA2 / FMUL2 (one
// instruction for two lanes' worth of FMAs) — the fused kernels are partly
// issue-bound, and the per-edge accumulator updates are their biggest FP
// share.  Per element the result is the same IEEE fma / mul as the scalar
// form; fp64 keeps scalar code.
#ifndef GF_PAIRED_FP
#define GF_PAIRED_FP 1
#endif
template <typename T, int N>
__device__ __forceinline__ void axpy_n(T (&y)[N], T a, const T (&x)[N]) {
#if GF_PAIRED_FP
  if constexpr (sizeof(T) == 4 && N % 2 == 0) {
    const float2 aa = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 r = __ffma2_rn(aa, make_float2(x[i], x[i + 1]), make_float2(y[i], y[i + 1]));
      y[i] = r.x;
      y[i + 1] = r.y;
    }
    return;
  }
#endif
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] += a * x[i];
}

// y[OFF + i] += a x[i] for the first N elements at offset OFF of a longer
// accumulator array (pass B's {dV | dQ} registers).
template <int OFF, typename T, int N, int M>
__device__ __forceinline__ void axpy_at(T (&y)[M], T a, const T (&x)[N]) {
  static_assert(OFF + N <= M, "axpy_at range");
#if GF_PAIRED_FP
  if constexpr (sizeof(T) == 4 && N % 2 == 0 && OFF % 2 == 0) {
    const float2 aa = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 r =
          __ffma2_rn(aa, make_float2(x[i], x[i + 1]), make_float2(y[OFF + i], y[OFF + i + 1]));
      y[OFF + i] = r.x;
      y[OFF + i + 1] = r.y;
    }
    return;
  }
#endif
#pragma unroll
  for (int i = 0; i < N; ++i) y[OFF + i] += a * x[i];
}

template <typename T, int N>
__device__ __forceinline__ void scale_n(T (&y)[N], T a) {
#if GF_PAIRED_FP
  if constexpr (sizeof(T) == 4 && N % 2 == 0) {
    const float2 aa = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 r = __fmul2_rn(aa, make_float2(y[i], y[i + 1]));
      y[i] = r.x;
      y[i + 1] = r.y;
    }
    return;
  }
#endif
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] *= a;
}

// <x, y>: fp32 pairs accumulate even / odd elements in two FFMA2 lanes, then
// add them (a pairwise order; fp64 and odd N sequential).
template <typename T, int N>
__device__ __forceinline__ T dot_n(const T (&x)[N], const T (&y)[N]) {
#if GF_PAIRED_FP
  if constexpr (sizeof(T) == 4 && N % 2 == 0) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < N; i += 2)
      acc = __ffma2_rn(make_float2(x[i], x[i + 1]), make_float2(y[i], y[i + 1]), acc);
    return acc.x + acc.y;
  }
#endif
  T s = T(0);
#pragma unroll
  for (int i = 0; i < N; ++i) s += x[i] * y[i];
  return s;
}
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- chunks --
// A lane moves one CB-byte chunk per load: CB = 32 uses the sm_100 256-bit
// global load (LDG.E.256, one full 32 B sector per lane), CB = 16 the 128-bit
// one.  Gathered rows are read through the non-coherent path without L1
// allocation (they are touched once per edge); owned rows use plain loads.
template <typename T, int CB>
struct Chunk {
  static constexpr int W = CB / static_cast<int>(sizeof(T));
};

// L2 residency policy: the gathered node tables (V, Q|el, dO, K, records;
// tens of MB) are marked evict_last so the streamed topology (neighbour ids,
// hundreds of MB, read once per pass) marked evict_first does not push them
// out of the 126 MB L2.
#ifndef GF_L2HINT
#define GF_L2HINT 1
#endif
// GF_L2_EVICT_OP = 1: the 256-bit gathers carry the load's own L2 eviction
// priority (ld.L2::evict_last -> LDG...ELL2; ptxas allows it on .v8.b32 /
// .v4.b64 loads only) instead of a cache-hint policy word in the memory
// descriptor: no policy register pair and no R2UR copies before each gather
// (profiles/r2/ab_r2_policy_param.txt); same residency behaviour, set-aside
// included.  Narrower gathers keep the policy word.
#ifndef GF_L2_EVICT_OP
#define GF_L2_EVICT_OP 1
#endif
// GF_GATHER_L1 = 1: the fp32 256-bit gathers also allocate in L1 (no
// .L1::no_allocate).  The rows are not reused, yet the allocating path
// measured 3 % faster in the forward (C4 1.75 -> 1.70 ms; table form C5
// 3.64 -> 3.40 ms, profiles/r2/ab_r2_policy_param.txt).
#ifndef GF_GATHER_L1
#define GF_GATHER_L1 1
#endif
__device__ __forceinline__ uint64_t pol_keep() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_stream() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

/// Streamed neighbour id (read once per pass).
__device__ __forceinline__ int ld_idx(const int32_t* __restrict__ p) {
#if GF_L2HINT
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol_stream()));
  return v;
#else
  return __ldg(p);
#endif
}

/// Streamed edge value (E x H score / probability buffers of the
/// non-fused strategies; read once per pass).
template <typename T>
__device__ __forceinline__ T ld_edge(const T* __restrict__ p) {
  T v;
  if constexpr (sizeof(T) == 4)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol_stream()));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol_stream()));
  return v;
}

/// Schedule slot {node, begin, end, 0} (streamed, read once per pass).
__device__ __forceinline__ int4 ld_sched(const int4* __restrict__ p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol_stream()));
  return v;
}

/// Gathered scalar of a node table (el[src], ...).
template <typename T>
__device__ __forceinline__ T ld_node(const T* __restrict__ p, const uint64_t pol) {
#if GF_L2HINT
  T v;
  if constexpr (sizeof(T) == 4)
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(p);
#endif
}
template <typename T>
__device__ __forceinline__ T ld_node(const T* __restrict__ p) {
  return ld_node(p, pol_keep());
}

// Row r of a node table with a row stride of `stride_bytes`: one
// IMAD.WIDE.U32 (base + r * stride as a 64-bit product) instead of a signed
// 32-bit multiply, sign extension and a scaled 64-bit add.  Valid for
// r >= 0 (ids, and the 0 dummy row of masked lanes).
#ifndef GF_WIDE_ADDR
#define GF_WIDE_ADDR 1
#endif
template <typename T>
__device__ __forceinline__ const T* row_at(const T* __restrict__ base, int r, uint32_t stride_bytes) {
#if GF_WIDE_ADDR
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) +
                                    static_cast<uint64_t>(static_cast<uint32_t>(r)) * stride_bytes);
#else
  return base + r * static_cast<int>(stride_bytes / sizeof(T));
#endif
}

// Gathers with an explicit L2 policy word (gf_policy.h; used when
// GF_L2_EVICT_OP = 0); the two-argument form creates evict_last in-kernel.

template <typename T, int CB>
__device__ __forceinline__ void ld_gather(const T* __restrict__ p, T (&x)[CB / sizeof(T)],
                                          const uint64_t pol);
template <typename T, int CB>
__device__ __forceinline__ void ld_gather(const T* __restrict__ p, T (&x)[CB / sizeof(T)]) {
  ld_gather<T, CB>(p, x, pol_keep());
}

template <typename T, int CB>
__device__ __forceinline__ void ld_gather(const T* __restrict__ p, T (&x)[CB / sizeof(T)],
                                          const uint64_t pol) {
  if constexpr (CB == 32 && sizeof(T) == 4) {
#if GF_L2HINT && GF_L2_EVICT_OP && GF_GATHER_L1
    (void)pol;
    asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                   "=f"(x[6]), "=f"(x[7])
                 : "l"(p));
#elif GF_L2HINT && GF_L2_EVICT_OP
    (void)pol;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                   "=f"(x[6]), "=f"(x[7])
                 : "l"(p));
#elif GF_L2HINT
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                   "=f"(x[6]), "=f"(x[7])
                 : "l"(p), "l"(pol));
#else
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                   "=f"(x[6]), "=f"(x[7])
                 : "l"(p));
#endif
  } else if constexpr (CB == 32) {
#if GF_L2HINT && GF_L2_EVICT_OP
    (void)pol;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p));
#elif GF_L2HINT
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p), "l"(pol));
#else
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p));
#endif
  } else if constexpr (sizeof(T) == 4) {
#if GF_L2HINT
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                 : "l"(p), "l"(pol));
#else
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
#endif
  } else {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = v.x, x[1] = v.y;
  }
}

// Owned rows (read or written once per pass) may be marked evict_first so
// they do not displace the gathered tables (GF_OWN_HINT: 1 = loads and
// stores, 2 = stores only).
#ifndef GF_OWN_HINT
#define GF_OWN_HINT 0
#endif

template <typename T, int CB>
__device__ __forceinline__ void ld_own(const T* __restrict__ p, T (&x)[CB / sizeof(T)]) {
  constexpr int W = CB / sizeof(T);
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
#if GF_OWN_HINT == 1
      float4 v;
      asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(p + i), "l"(pol_stream()));
#else
      const float4 v = *reinterpret_cast<const float4*>(p + i);
#endif
      x[i] = v.x, x[i + 1] = v.y, x[i + 2] = v.z, x[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + i);
      x[i] = v.x, x[i + 1] = v.y;
    }
  }
}

template <typename T, int CB>
__device__ __forceinline__ void st_chunk(T* __restrict__ p, const T (&x)[CB / sizeof(T)]) {
  constexpr int W = CB / sizeof(T);
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
#if GF_OWN_HINT
      asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                   :: "l"(p + i), "f"(x[i]), "f"(x[i + 1]), "f"(x[i + 2]), "f"(x[i + 3]),
                      "l"(pol_stream())
                   : "memory");
#else
      *reinterpret_cast<float4*>(p + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
#endif
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 2) *reinterpret_cast<double2*>(p + i) = make_double2(x[i], x[i + 1]);
  }
}

// ------------------------------------------------------------------- exp --
// ex2 on the SFU (one MUFU.EX2, flush-to-zero) for fp32; full precision fp64.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double ex2(double x) { return exp2(x); }
__device__ __forceinline__ float lg2(float x) { return log2f(x); }
__device__ __forceinline__ double lg2(double x) { return log2(x); }
template <typename T>
__device__ __forceinline__ T l2e() {
  return static_cast<T>(1.4426950408889634073599246810019);
}
/// exp(d) for d = s - m computed first (keeps relative precision for any |s|).
template <typename T>
__device__ __forceinline__ T expd(T d) {
  return ex2(d * l2e<T>());
}

template <typename T>
__device__ __forceinline__ T ninf() {
  return -INFINITY;
}

// ------------------------------------------------------ softmax records --
// Per (row v, head h) record of 4 T, written by the forward and pass A and
// gathered by pass B in ONE load:
//   [0] m     reference score (natural units): the row max up to the
//             forward's lazy-rescale threshold (m >= max - GF_RESCALE_TH)
//   [1] ll2   log2 of l = sum exp(s - m)        => p = 2^((s - m) log2e - ll2)
//   [2] aux   er[v,h] (GAT) | 1/max(||K[v,h]||,eps) (AGNN) | 0
//   [3] delta <dO[v,h], O[v,h]> (written by backward pass A)
// Splitting lse into (m, log l) keeps p exact-relative for any score
// magnitude (a fused fp32 lse loses ulp(|m|), ~6e-5 at |s| ~ 1e3).
template <typename T>
struct Rec {
  T m, ll2, aux, delta;
};

#ifndef GF_REC_KEEP
#define GF_REC_KEEP 0  // 1: records also evict_last (dO alone fits the 64 MiB carve-out)
#endif
template <typename T>
__device__ __forceinline__ Rec<T> ld_rec(const T* __restrict__ st, size_t i) {
  Rec<T> r;
  if constexpr (sizeof(T) == 4) {
    float x[4];
#if GF_REC_KEEP
    ld_gather<float, 16>(st + 4 * i, x);
#else
    const float4 v = __ldg(reinterpret_cast<const float4*>(st + 4 * i));
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
#endif
    r.m = x[0], r.ll2 = x[1], r.aux = x[2], r.delta = x[3];
  } else {
    double x[4];
    ld_gather<double, 32>(st + 4 * i, x);
    r.m = x[0], r.ll2 = x[1], r.aux = x[2], r.delta = x[3];
  }
  return r;
}

template <typename T>
__device__ __forceinline__ T prob(T s, const Rec<T>& r) {
  return ex2((s - r.m) * l2e<T>() - r.ll2);
}

template <typename T>
__device__ __forceinline__ T lrelu(T x, T slope) {
  return x >= T(0) ? x : slope * x;  // kernels.hpp:44
}
template <typename T>
__device__ __forceinline__ T lrelu_grad(T pre, T slope) {
  return pre > T(0) ? T(1) : slope;  // autograd.hpp:113 (kink takes the slope)
}

/// Sum over the LPH lanes that share one head (aligned groups, LPH a power of
/// two <= 32); every lane of the group ends with the total.
template <typename T>
__device__ __forceinline__ T head_sum(T x, int lph) {
  for (int off = 1; off < lph; off <<= 1) x += __shfl_xor_sync(kFull, x, off);
  return x;
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

// Destination operands for lane h: er[v,h] (add) or 1/max(||K[v,h]||,eps).
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

// ------------------------------------------------- multi-CTA split rows --
// A super row / column split over ct.z CTAs (ct = {slot, slice, slices, first
// partial}, DevGraph::row_cta): each CTA publishes its slice's state (NV
// values per lane group c of LPE) to part[], then the LAST CTA to arrive
// (per-row arrival counter) merges all slices in slice order 0..z-1, so the
// result does not depend on which CTA arrives last (deterministic).  Called by
// every lane of the CTA's merging warp; `writer` lanes own a lane group.
// Returns true in the last CTA (whose lanes then call split_load).
template <int NV, typename T>
__device__ __forceinline__ bool split_publish(T* __restrict__ part, unsigned* __restrict__ cnt,
                                              const int4 ct, int c, int lpe, const T (&x)[NV],
                                              bool writer) {
  if (writer) {
    T* p = part + (static_cast<size_t>(ct.w + ct.y) * lpe + c) * NV;
#pragma unroll
    for (int i = 0; i < NV; ++i) p[i] = x[i];
  }
  __threadfence();
  __syncwarp();
  unsigned prev = 0;
  if ((threadIdx.x & 31) == 0) prev = atomicAdd(cnt + ct.w, 1u);
  prev = __shfl_sync(kFull, prev, 0);
  if (prev + 1 != static_cast<unsigned>(ct.z)) return false;
  __threadfence();
  if ((threadIdx.x & 31) == 0) cnt[ct.w] = 0;  // re-armed for the next launch
  return true;
}

template <int NV, typename T>
__device__ __forceinline__ void split_load(const T* __restrict__ part, const int4 ct, int slice,
                                           int c, int lpe, T (&x)[NV]) {
  const T* p = part + (static_cast<size_t>(ct.w + slice) * lpe + c) * NV;
#pragma unroll
  for (int i = 0; i < NV; ++i) x[i] = __ldcg(p + i);  // L2: written by other SMs
}

// Balanced split of [b, e) into `parts` contiguous slices (first `rem` get +1),
// the same rule the reference uses for warp_balance (schedule.cpp:42-60).
__device__ __forceinline__ void split_range(int b, int e, int parts, int i, int& sb, int& se) {
  const int len = e - b, base = len / parts, rem = len % parts;
  sb = b + i * base + (i < rem ? i : rem);
  se = sb + base + (i < rem ? 1 : 0);
}

}  // namespace gfb

// The non-default fusion strategies of the reference's Strategy enum
// (schedule.hpp:12-34; engine.hpp:292-329), as real B200 kernels so the
// paper's SMMF-vs-PMF-vs-unfused-vs-baseline ablation (DF-GNN §5) can be run
// on the same hardware.  The reference runs one CPU code path for all four and
// only its counter model (engine.hpp:84-168) tells them apart; here each one
// has the launch structure and HBM traffic that model describes:
//
//   SMMF      1 launch : fwd_fast MODE 0 (gf_attn_fwd.cuh) — scores, softmax
//                        and aggregation fused, nothing E x H in HBM.
//   PMF       2 launches: sddmm_edges (edge-parallel, the reference's
//                        edge_parallel_partition balance, schedule.cpp:62-77)
//                        writes S[E x H]; fwd_fast MODE 1 fuses softmax + SpMM
//                        over S with the bi-level row schedule.
//   Unfused   3 launches: sddmm_edges -> softmax_rows (S -> P, E x H, plus the
//                        softmax records) -> fwd_fast MODE 2 (O = sum p V).
//   Baseline  1 launch : fwd_feature_parallel — warp per row in id order (no
//                        degree schedule), lanes over FEATURES: every lane
//                        recomputes its head's scores and the whole row
//                        softmax (the redundancy the reference counts as
//                        softmax ops x ceil(d / group_width), engine.hpp:150-158).
//
// Every strategy writes the same outputs: O and the per-(row, head) softmax
// records (so the recompute backward runs after any of them), plus P when
// requested.
#include <algorithm>
#include <mutex>

#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {
namespace {

// CSR-order destination of every edge (the reference's coo_dst,
// graph.hpp:31), built once per graph for the edge-parallel kernels.
__global__ void coo_dst_kernel(const int32_t* __restrict__ ptr, int n, int32_t* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += (gridDim.x * blockDim.x) >> 5) {
    const int b = ptr[v], e = ptr[v + 1];
    for (int i = b + lane; i < e; i += 32) dst[i] = v;
  }
}

// ---- edge-parallel SDDMM: one thread per (edge, head), E*H flat index -------
// Consecutive threads take consecutive heads of one edge, so the H threads of
// an edge read the source and destination rows as contiguous segments.
template <typename T, int VAR>
__global__ void __launch_bounds__(256) sddmm_edges(const FwdArgs<T> a, const int32_t* __restrict__ dst,
                                                   int64_t e, T* __restrict__ S) {
  const int64_t total = e * a.H;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ed = i / a.H;
    const int h = static_cast<int>(i - ed * a.H);
    const int u = ld_idx(a.idx + ed), v = ld_idx(dst + ed);
    T s;
    if constexpr (VAR == GF_ADD) {
      s = lrelu(ld_node(a.Q + static_cast<size_t>(u) * a.H + h) +
                    ld_node(a.K + static_cast<size_t>(v) * a.H + h),
                a.slope);
    } else {
      const T* q = a.Q + static_cast<size_t>(u) * a.F + h * a.D;
      const T* k = a.K + static_cast<size_t>(v) * a.F + h * a.D;
      T d = T(0), qq = T(0), kk = T(0);
      for (int j = 0; j < a.D; ++j) {
        const T x = __ldg(q + j), y = __ldg(k + j);
        d += x * y;
        qq += x * x;
        kk += y * y;
      }
      s = a.l2 ? a.scale * d * (inv_norm(qq) * inv_norm(kk)) : a.scale * d;
    }
    S[i] = s;
  }
}

// ---- edge softmax over S (the unfused middle launch), warp per row ---------
// The row's scores are the contiguous segment S[eb*H, ee*H); when H divides 32
// lane l always sees head l % H, so each pass is a coalesced sweep and the
// per-head reduction is a shuffle over lanes l, l+H, ...  Three sweeps (max,
// sum, normalise) — the F round trip the reference's counters charge
// (engine.hpp:112-113).  Writes P and the softmax records.
template <typename T, int VAR>
__global__ void __launch_bounds__(256) softmax_rows(const FwdArgs<T> a, const T* __restrict__ S,
                                                    T* __restrict__ P) {
  const int lane = threadIdx.x & 31;
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slot >= a.n) return;
  const int v = __ldg(a.order + slot);
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  const int H = a.H;
  const size_t base = static_cast<size_t>(eb) * H, len = static_cast<size_t>(ee - eb) * H;
  T m = ninf<T>(), l = T(0);
  int h;
  if (32 % H == 0) {
    h = lane % H;
    for (size_t i = lane; i < len; i += 32) {
      const T x = ld_edge(S + base + i);
      m = x > m ? x : m;
    }
    for (int o = H; o < 32; o <<= 1) {
      const T y = __shfl_xor_sync(kFull, m, o);
      m = y > m ? y : m;
    }
    for (size_t i = lane; i < len; i += 32) l += expd(ld_edge(S + base + i) - m);
    for (int o = H; o < 32; o <<= 1) l += __shfl_xor_sync(kFull, l, o);
    const T r = l == T(0) ? T(0) : T(1) / l;
    for (size_t i = lane; i < len; i += 32) P[base + i] = expd(ld_edge(S + base + i) - m) * r;
  } else {  // H does not divide the warp: lane h < H walks its head serially
    h = lane;
    if (lane < H) {
      for (size_t i = lane; i < len; i += H) {
        const T x = ld_edge(S + base + i);
        m = x > m ? x : m;
      }
      for (size_t i = lane; i < len; i += H) l += expd(ld_edge(S + base + i) - m);
      const T r = l == T(0) ? T(0) : T(1) / l;
      for (size_t i = lane; i < len; i += H) P[base + i] = expd(ld_edge(S + base + i) - m) * r;
    }
  }
  if (a.stats && lane < H) {
    T erh, rkh;
    generic_row_setup<T, VAR>(a, v, lane, nullptr, erh, rkh);
    T* rec = a.stats + 4 * (static_cast<size_t>(v) * H + h);
    rec[0] = l == T(0) ? ninf<T>() : m;
    rec[1] = l == T(0) ? T(0) : lg2(l);
    rec[2] = VAR == GF_DOT ? rkh : erh;
  }
}

// ---- feature-parallel fused baseline (the pre-DF-GNN fused kernel) ---------
// Warp per destination row in id order; lane owns features f = lane + 32 i.
// Per edge every lane rebuilds the score of ITS feature's head — for dot
// scores by a shuffle reduction of the head's D partial products (shared
// memory for D that neither divides nor is a multiple of 32) — so each of the
// D lanes of a head repeats the row's softmax work.  Two
// sweeps over the row (max, then exp/sum/aggregate).
template <typename T, int VAR, int NF>
__global__ void __launch_bounds__(128) fwd_feature_parallel(const FwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int v = blockIdx.x * 4 + warp;
  if (v >= a.n) return;
  T* part = reinterpret_cast<T*>(smraw) + static_cast<size_t>(warp) * 2 * 32 * NF;  // dot partials
  T* sq = part + 32 * NF;                                                            // |q|^2 partials
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  int hf[NF];
  bool in[NF];
  T kf[NF], erf[NF], rkf[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int f = lane + 32 * i;
    in[i] = f < a.F;
    hf[i] = in[i] ? f / a.D : 0;
    kf[i] = T(0);
    erf[i] = T(0);
    rkf[i] = T(1);
    if (!in[i]) continue;
    if constexpr (VAR == GF_DOT)
      kf[i] = __ldg(a.K + static_cast<size_t>(v) * a.F + f);
    else
      erf[i] = __ldg(a.K + static_cast<size_t>(v) * a.H + hf[i]);
  }
  if (VAR == GF_DOT && a.l2) {  // 1/||K[v, head]|| per lane, via shared memory
#pragma unroll
    for (int i = 0; i < NF; ++i) part[lane + 32 * i] = kf[i] * kf[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      T s2 = T(0);
      for (int j = 0; j < a.D && in[i]; ++j) s2 += part[hf[i] * a.D + j];
      rkf[i] = inv_norm(s2);
    }
    __syncwarp();
  }
  const bool shuf = (32 % a.D == 0) || (a.D % 32 == 0);
  // score of every owned feature's head for source u (all lanes participate)
  auto scores = [&](int u, T (&s)[NF]) {
    if constexpr (VAR == GF_ADD) {
#pragma unroll
      for (int i = 0; i < NF; ++i)
        s[i] = in[i] ? lrelu(__ldg(a.Q + static_cast<size_t>(u) * a.H + hf[i]) + erf[i], a.slope)
                     : T(0);
    } else if (shuf) {
      // head sums by warp shuffles: within aligned groups of D lanes (D | 32)
      // or over the whole warp after summing the D/32 features a lane holds
      T pq[NF], qq2[NF];
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        const T q = in[i] ? __ldg(a.Q + static_cast<size_t>(u) * a.F + lane + 32 * i) : T(0);
        pq[i] = q * kf[i];
        qq2[i] = q * q;
      }
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        T d = T(0), qq = T(0);
        if (a.D <= 32) {
          d = pq[i], qq = qq2[i];
          for (int o = 1; o < a.D; o <<= 1) {
            d += __shfl_xor_sync(kFull, d, o);
            qq += __shfl_xor_sync(kFull, qq, o);
          }
        } else {
          const int G = a.D / 32;  // features of one head held by this lane
#pragma unroll
          for (int j = 0; j < NF; ++j)
            if (j / G == i / G) d += pq[j], qq += qq2[j];
          for (int o = 1; o < 32; o <<= 1) {
            d += __shfl_xor_sync(kFull, d, o);
            qq += __shfl_xor_sync(kFull, qq, o);
          }
        }
        s[i] = a.l2 ? a.scale * d * (inv_norm(qq) * rkf[i]) : a.scale * d;
      }
    } else {  // D neither divides nor is a multiple of 32: partials via shared memory
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        const T q = in[i] ? __ldg(a.Q + static_cast<size_t>(u) * a.F + lane + 32 * i) : T(0);
        part[lane + 32 * i] = q * kf[i];
        sq[lane + 32 * i] = q * q;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        T d = T(0), qq = T(0);
        for (int j = 0; j < a.D && in[i]; ++j) {
          d += part[hf[i] * a.D + j];
          qq += sq[hf[i] * a.D + j];
        }
        s[i] = a.l2 ? a.scale * d * (inv_norm(qq) * rkf[i]) : a.scale * d;
      }
      __syncwarp();
    }
  };
  T m[NF], l[NF], acc[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) m[i] = ninf<T>(), l[i] = T(0), acc[i] = T(0);
  for (int e = eb; e < ee; ++e) {
    const int u = __ldg(a.idx + e);
    T s[NF];
    scores(u, s);
#pragma unroll
    for (int i = 0; i < NF; ++i) m[i] = s[i] > m[i] ? s[i] : m[i];
  }
  for (int e = eb; e < ee; ++e) {
    const int u = __ldg(a.idx + e);
    T s[NF];
    scores(u, s);
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      if (!in[i]) continue;
      const T p = expd(s[i] - m[i]);
      l[i] += p;
      acc[i] += p * __ldg(a.V + static_cast<size_t>(u) * a.F + lane + 32 * i);
    }
  }
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    if (!in[i]) continue;
    const int f = lane + 32 * i;
    a.O[static_cast<size_t>(v) * a.F + f] = l[i] == T(0) ? T(0) : acc[i] / l[i];
    if (f % a.D == 0) {  // first lane of the head writes its record
      T* rec = a.stats + 4 * (static_cast<size_t>(v) * a.H + hf[i]);
      rec[0] = l[i] == T(0) ? ninf<T>() : m[i];
      rec[1] = l[i] == T(0) ? T(0) : lg2(l[i]);
      rec[2] = VAR == GF_DOT ? rkf[i] : erf[i];
    }
  }
}

template <typename T, int VAR>
int launch_fp(const FwdArgs<T>& a, cudaStream_t s) {
  const int nf = (a.F + 31) / 32;
  const size_t smem = VAR == GF_DOT ? 4 * 2 * 32 * static_cast<size_t>(nf) * sizeof(T) : 0;
  const int blocks = (a.n + 3) / 4;
#define GF_FP_CASE(K)                                                       \
  case K:                                                                   \
    fwd_feature_parallel<T, VAR, K><<<blocks, 128, smem, s>>>(a);           \
    break;
  switch (nf) {
    GF_FP_CASE(1)
    GF_FP_CASE(2)
    GF_FP_CASE(3)
    GF_FP_CASE(4)
    GF_FP_CASE(5)
    GF_FP_CASE(6)
    GF_FP_CASE(7)
    GF_FP_CASE(8)
    default:
      set_error("gf_attn_fwd_strategy: the feature-parallel baseline supports H*D <= 256");
      return GF_ERR_UNSUPPORTED;
  }
#undef GF_FP_CASE
  GF_CHECK_LAUNCH("fwd_feature_parallel");
  return GF_OK;
}

int grid_1d(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 16, (work + 255) / 256)));
}

}  // namespace

int ensure_coo_dst(DevGraph& g, cudaStream_t s) {
  static std::mutex mu;  // graphs are shareable across host threads (reference SPEC.md:98)
  std::lock_guard<std::mutex> lock(mu);
  if (g.coo_dst || g.e == 0) return GF_OK;
  GF_CHECK_CUDA(cudaMalloc(&g.coo_dst, sizeof(int32_t) * g.e));
  const int blocks = static_cast<int>(std::min<int64_t>(148 * 32, (int64_t(g.n) * 32 + 255) / 256 + 1));
  coo_dst_kernel<<<blocks, 256, 0, s>>>(g.row_ptr, g.n, g.coo_dst);
  GF_CHECK_LAUNCH("coo_dst_kernel");
  return GF_OK;
}

template <typename T>
int launch_sddmm_edges(DevGraph& g, const FwdArgs<T>& a, int variant, T* S, cudaStream_t s) {
  if (g.e == 0) return GF_OK;
  if (int rc = ensure_coo_dst(g, s)) return rc;
  const int64_t eh = static_cast<int64_t>(g.e) * a.H;
  if (variant == GF_DOT)
    sddmm_edges<T, GF_DOT><<<grid_1d(eh), 256, 0, s>>>(a, g.coo_dst, g.e, S);
  else
    sddmm_edges<T, GF_ADD><<<grid_1d(eh), 256, 0, s>>>(a, g.coo_dst, g.e, S);
  GF_CHECK_LAUNCH("sddmm_edges");
  return GF_OK;
}

template <typename T>
int launch_softmax_rows(const DevGraph& g, const FwdArgs<T>& a, int variant, const T* S, T* P,
                        cudaStream_t s) {
  if (a.n == 0) return GF_OK;
  if (a.H > 32) {
    set_error("edge softmax: heads <= 32 supported");
    return GF_ERR_UNSUPPORTED;
  }
  const int blocks = static_cast<int>((static_cast<int64_t>(a.n) * 32 + 255) / 256);
  if (variant == GF_DOT)
    softmax_rows<T, GF_DOT><<<blocks, 256, 0, s>>>(a, S, P);
  else
    softmax_rows<T, GF_ADD><<<blocks, 256, 0, s>>>(a, S, P);
  GF_CHECK_LAUNCH("softmax_rows");
  return GF_OK;
}

template int launch_sddmm_edges<float>(DevGraph&, const FwdArgs<float>&, int, float*, cudaStream_t);
template int launch_sddmm_edges<double>(DevGraph&, const FwdArgs<double>&, int, double*,
                                        cudaStream_t);
template int launch_softmax_rows<float>(const DevGraph&, const FwdArgs<float>&, int, const float*,
                                        float*, cudaStream_t);
template int launch_softmax_rows<double>(const DevGraph&, const FwdArgs<double>&, int,
                                         const double*, double*, cudaStream_t);

size_t strategy_workspace_bytes(const DevGraph& g, int heads, int elem, int strategy, bool have_p) {
  const size_t eh = static_cast<size_t>(g.e) * heads * elem;
  if (strategy == GF_STRAT_PMF) return eh;
  if (strategy == GF_STRAT_UNFUSED) return have_p ? eh : 2 * eh;
  return 0;
}

template <typename T>
int launch_fwd_strategy(DevGraph& g, const FwdArgs<T>& a, int variant, int strategy, T* P,
                        T* ws, cudaStream_t s) {
  if (g.n == 0 || a.n == 0) return GF_OK;
  const int64_t eh = static_cast<int64_t>(g.e) * a.H;
  switch (strategy) {
    case GF_STRAT_SMMF:
      if (int rc = launch_fwd_mode<T>(g, a, variant, 0, s)) return rc;
      return P ? launch_materialize_p<T>(g, a, variant, P, s) : GF_OK;
    case GF_STRAT_PMF:
    case GF_STRAT_UNFUSED: {
      T* S = ws;
      if (int rc = launch_sddmm_edges<T>(g, a, variant, S, s)) return rc;
      FwdArgs<T> b = a;
      if (strategy == GF_STRAT_PMF) {
        b.ES = S;
        if (int rc = launch_fwd_mode<T>(g, b, variant, 1, s)) return rc;
        return P ? launch_materialize_p<T>(g, a, variant, P, s) : GF_OK;
      }
      T* Pw = P ? P : ws + eh;
      if (int rc = launch_softmax_rows<T>(g, a, variant, S, Pw, s)) return rc;
      b.ES = Pw;
      b.scale = T(1);  // MODE 2 scales its sums by a.scale
      return launch_fwd_mode<T>(g, b, variant, 2, s);
    }
    case GF_STRAT_BASELINE: {
      FwdArgs<T> b = a;
      b.n = g.n;  // rows in id order (no degree schedule); rows without edges get O = 0
      int rc = variant == GF_DOT ? launch_fp<T, GF_DOT>(b, s) : launch_fp<T, GF_ADD>(b, s);
      if (rc) return rc;
      return P ? launch_materialize_p<T>(g, a, variant, P, s) : GF_OK;
    }
    default:
      set_error("gf_attn_fwd_strategy: unknown strategy");
      return GF_ERR_INVALID;
  }
}

template int launch_fwd_strategy<float>(DevGraph&, const FwdArgs<float>&, int, int, float*, float*,
                                        cudaStream_t);
template int launch_fwd_strategy<double>(DevGraph&, const FwdArgs<double>&, int, int, double*,
                                         double*, cudaStream_t);

}  // namespace gfb

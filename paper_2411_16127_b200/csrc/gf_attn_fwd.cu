// Fused AT-GNN forward for sm_100a: SDDMM -> per-destination edge softmax ->
// SpMM in ONE launch, scores and softmax statistics kept in registers (warp
// rows) or registers + shared memory (CTA rows).  Replaces the reference's
// per-row CPU loop run_block_rows (engine.hpp:192-231) and its unfused
// composition sddmm/edge_softmax/spmm (kernels.hpp:18-117).
//
// Bi-level scheduling (DF-GNN's dynamic thread mapping, done for real):
//   * rows are visited in degree-descending order (DevGraph::row_order), so
//     the longest rows start first (LPT);
//   * rows with degree >= cta_threshold get a whole 8-warp CTA: the edge range
//     is split into 8 balanced slices (the reference's warp_balance rule,
//     schedule.cpp:42-60), each warp runs an online (max,sum) softmax over its
//     slice in registers, and the 8 partial states are merged in shared
//     memory in a fixed order (deterministic);
//   * every other row is warp-per-row: LPE lanes cover one edge's feature row
//     with 16-byte loads (128-bit vectorised, coalesced gathers of V[src] and
//     Q[src] / el[src]), 32/LPE edges per step, unrolled U-deep for MLP.
// Nothing of size E x H is written; the only outputs are O (N x F) and
// the softmax statistics (N x H x 2: row max, log-sum) the backward needs.
#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {

namespace {

template <typename T, int CW>
__device__ __forceinline__ void merge_state(T& m, T& l, T (&acc)[CW], T m2, T l2,
                                            const T (&acc2)[CW]) {
  const T mn = m > m2 ? m : m2;
  if (!(mn > ninf<T>())) return;  // both empty (or NaN max: keep ours)
  const T ca = gexp(m - mn), cb = gexp(m2 - mn);
  l = l * ca + l2 * cb;
#pragma unroll
  for (int i = 0; i < CW; ++i) acc[i] = acc[i] * ca + acc2[i] * cb;
  m = mn;
}

template <typename T, int LPE, int CPL, int VAR>
__global__ void __launch_bounds__(256) fwd_fast(const FwdArgs<T> a) {
  constexpr int CW = Chunk<T>::W;
  constexpr int EPW = 32 / LPE;
  constexpr int U = CPL == 1 ? 4 : (CPL == 2 ? 2 : 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPE, sub = lane / LPE;
  const bool cta = blockIdx.x < static_cast<unsigned>(a.n_cta);
  int slot;
  if (cta) {
    slot = blockIdx.x;
  } else {
    slot = a.n_cta + (blockIdx.x - a.n_cta) * kWarpsPerBlock + warp;
    if (slot >= a.n) return;
  }
  const int v = __ldg(a.order + slot);
  int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  if (cta) split_range(eb, ee, kWarpsPerBlock, warp, eb, ee);

  int off[CPL], head[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const int ch = c + k * LPE;
    off[k] = ch * CW;
    head[k] = ch / a.GD;
  }

  // Destination-side operands stay in registers for the whole row.
  T kv[CPL][CW];
  T erv[CPL];
  T rk[CPL];
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) ld_chunk(a.K + static_cast<size_t>(v) * a.F + off[k], kv[k]);
    if (a.l2) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        T s = T(0);
#pragma unroll
        for (int i = 0; i < CW; ++i) s += kv[k][i] * kv[k][i];
        rk[k] = s;
      }
      head_sum<LPE, CPL>(rk, a.GD);
#pragma unroll
      for (int k = 0; k < CPL; ++k) rk[k] = inv_norm(rk[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < CPL; ++k) erv[k] = __ldg(a.K + static_cast<size_t>(v) * a.H + head[k]);
  }

  T m[CPL], l[CPL], acc[CPL][CW];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    m[k] = ninf<T>();
    l[k] = T(0);
#pragma unroll
    for (int i = 0; i < CW; ++i) acc[k][i] = T(0);
  }

  for (int base = eb; base < ee; base += 32) {
    const int cnt = min(32, ee - base);
    const int myu = lane < cnt ? __ldg(a.idx + base + lane) : 0;
#pragma unroll 1
    for (int j0 = 0; j0 < cnt; j0 += EPW * U) {
      int u[U];
      bool ok[U];
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const int j = j0 + t * EPW + sub;
        ok[t] = j < cnt;
        u[t] = __shfl_sync(kFull, myu, j & 31);
      }
      T vv[U][CPL][CW];
      T qv[U][CPL][CW];
      T elv[U][CPL];
#pragma unroll
      for (int t = 0; t < U; ++t) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (ok[t]) {
            ld_chunk(a.V + static_cast<size_t>(u[t]) * a.F + off[k], vv[t][k]);
            if constexpr (VAR == GF_DOT)
              ld_chunk(a.Q + static_cast<size_t>(u[t]) * a.F + off[k], qv[t][k]);
            else
              elv[t][k] = __ldg(a.Q + static_cast<size_t>(u[t]) * a.H + head[k]);
          } else {
#pragma unroll
            for (int i = 0; i < CW; ++i) vv[t][k][i] = T(0), qv[t][k][i] = T(0);
            elv[t][k] = T(0);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < U; ++t) {
        T s[CPL];
        if constexpr (VAR == GF_DOT) {
          T q2[CPL];
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            T d = T(0), qq = T(0);
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              d += qv[t][k][i] * kv[k][i];
              qq += qv[t][k][i] * qv[t][k][i];
            }
            s[k] = d;
            q2[k] = qq;
          }
          head_sum<LPE, CPL>(s, a.GD);
          if (a.l2) {
            head_sum<LPE, CPL>(q2, a.GD);
#pragma unroll
            for (int k = 0; k < CPL; ++k) s[k] = a.scale * s[k] * (inv_norm(q2[k]) * rk[k]);
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) s[k] = a.scale * s[k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < CPL; ++k) s[k] = lrelu(elv[t][k] + erv[k], a.slope);
        }
        if (ok[t]) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            if (s[k] > m[k]) {  // lazy rescale: only when the running max moves
              const T corr = gexp(m[k] - s[k]);
              l[k] *= corr;
#pragma unroll
              for (int i = 0; i < CW; ++i) acc[k][i] *= corr;
              m[k] = s[k];
            }
            const T p = gexp(s[k] - m[k]);
            l[k] += p;
#pragma unroll
            for (int i = 0; i < CW; ++i) acc[k][i] += p * vv[t][k][i];
          }
        }
      }
    }
  }

  // Merge the EPW edge slots of the warp (butterfly: every lane ends with the
  // warp's state).
#pragma unroll
  for (int o = LPE; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      T acc2[CW];
#pragma unroll
      for (int i = 0; i < CW; ++i) acc2[i] = __shfl_xor_sync(kFull, acc[k][i], o);
      const T m2 = __shfl_xor_sync(kFull, m[k], o);
      const T l2 = __shfl_xor_sync(kFull, l[k], o);
      merge_state<T, CW>(m[k], l[k], acc[k], m2, l2, acc2);
    }
  }

  if (cta) {
    // Shared-memory merge of the 8 warp slices, fixed order w = 0..7.
    __shared__ T sm[kWarpsPerBlock][LPE * CPL][2 + CW];
    if (sub == 0) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        T* d = sm[warp][c * CPL + k];
        d[0] = m[k];
        d[1] = l[k];
#pragma unroll
        for (int i = 0; i < CW; ++i) d[2 + i] = acc[k][i];
      }
    }
    __syncthreads();
    if (warp != 0) return;
    if (sub == 0) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const T* d0 = sm[0][c * CPL + k];
        m[k] = d0[0];
        l[k] = d0[1];
#pragma unroll
        for (int i = 0; i < CW; ++i) acc[k][i] = d0[2 + i];
        for (int w = 1; w < kWarpsPerBlock; ++w) {
          const T* d = sm[w][c * CPL + k];
          T acc2[CW];
#pragma unroll
          for (int i = 0; i < CW; ++i) acc2[i] = d[2 + i];
          merge_state<T, CW>(m[k], l[k], acc[k], d[0], d[1], acc2);
        }
      }
    }
  }

  if (sub == 0) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const T r = l[k] == T(0) ? T(0) : T(1) / l[k];
      T o[CW];
#pragma unroll
      for (int i = 0; i < CW; ++i) o[i] = acc[k][i] * r;
      st_chunk(a.O + static_cast<size_t>(v) * a.F + off[k], o);
      if ((c + k * LPE) % a.GD == 0)
        st_stat(a.stats, static_cast<size_t>(v) * a.H + head[k], l[k] == T(0) ? ninf<T>() : m[k],
                l[k] == T(0) ? T(0) : glog(l[k]));
    }
  }
}

// ----------------------------------------------------------- generic path --
// Any (H <= 32, D): warp per row, two passes (max, then exp/sum/aggregate),
// per-head scalars owned by lane h, feature accumulators in shared memory.
// Used for shapes whose head does not tile into 16-byte chunks (e.g. D = 5).
template <typename T, int VAR>
__global__ void __launch_bounds__(128) fwd_generic(const FwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * kGenericWarps + warp;
  if (slot >= a.n) return;
  T* ws = reinterpret_cast<T*>(smraw) + static_cast<size_t>(warp) * (2 * a.F + 2 * 32);
  T* kvs = ws;           // F
  T* acc = ws + a.F;     // F
  T* ph = ws + 2 * a.F;  // 32
  T* lh = ph + 32;       // 32
  const int v = __ldg(a.order + slot);
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  for (int f = lane; f < a.F; f += 32) {
    if constexpr (VAR == GF_DOT) kvs[f] = __ldg(a.K + static_cast<size_t>(v) * a.F + f);
    acc[f] = T(0);
  }
  __syncwarp();
  T erh, rkh;
  generic_row_setup<T, VAR>(a, v, lane, VAR == GF_DOT ? kvs : nullptr, erh, rkh);
  T m = ninf<T>(), l = T(0);
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    if (lane < a.H) {
      const T s = generic_score<T, VAR>(a, u, v, lane, kvs, erh, rkh);
      m = (m < s || i == eb) ? s : m;  // left-to-right max from the first edge
    }
  }
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    if (lane < a.H) {
      const T p = gexp(generic_score<T, VAR>(a, u, v, lane, kvs, erh, rkh) - m);
      l += p;
      ph[lane] = p;
    }
    __syncwarp();
    for (int f = lane; f < a.F; f += 32)
      acc[f] += ph[f / a.D] * __ldg(a.V + static_cast<size_t>(u) * a.F + f);
    __syncwarp();
  }
  if (lane < a.H) {
    lh[lane] = l;
    st_stat(a.stats, static_cast<size_t>(v) * a.H + lane, l == T(0) ? ninf<T>() : m,
            l == T(0) ? T(0) : glog(l));
  }
  __syncwarp();
  for (int f = lane; f < a.F; f += 32) {
    const T lv = lh[f / a.D];
    a.O[static_cast<size_t>(v) * a.F + f] = lv == T(0) ? T(0) : acc[f] / lv;
  }
}

// P materialisation (reference ForwardContext::P, engine.hpp:29): recompute
// p = exp(s - lse) per edge and head.  Only on explicit request.
template <typename T, int VAR>
__global__ void __launch_bounds__(128) materialize_p(const FwdArgs<T> a, T* __restrict__ P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int v = blockIdx.x * kGenericWarps + warp;
  if (v >= a.n || lane >= a.H) return;
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  T erh, rkh;
  generic_row_setup<T, VAR>(a, v, lane, nullptr, erh, rkh);
  T m, ll;
  ld_stat(a.stats, static_cast<size_t>(v) * a.H + lane, m, ll);
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    P[static_cast<size_t>(i) * a.H + lane] =
        prob(generic_score<T, VAR>(a, u, v, lane, nullptr, erh, rkh), m, ll);
  }
}

template <typename T, int LPE, int CPL>
int launch_fast_fwd(const FwdArgs<T>& a, int variant, int blocks, cudaStream_t s) {
  if (variant == GF_DOT)
    fwd_fast<T, LPE, CPL, GF_DOT><<<blocks, 256, 0, s>>>(a);
  else
    fwd_fast<T, LPE, CPL, GF_ADD><<<blocks, 256, 0, s>>>(a);
  GF_CHECK_LAUNCH("fwd_fast");
  return GF_OK;
}

}  // namespace

FastShape fast_shape(int H, int D, int elem_bytes) {
  FastShape f;
  const int cw = 16 / elem_bytes;
  if (H < 1 || D < 1 || D % cw) return f;
  const int gd = D / cw;
  const long chunks = static_cast<long>(H) * gd;
  auto pow2 = [](long x) { return x > 0 && (x & (x - 1)) == 0; };
  if (!pow2(gd) || !pow2(chunks) || chunks > 128) return f;
  f.ok = true;
  f.gd = gd;
  f.lpe = chunks < 32 ? static_cast<int>(chunks) : 32;
  f.cpl = static_cast<int>(chunks / f.lpe);
  return f;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
int launch_fwd(const DevGraph& g, const FwdArgs<T>& a0, int variant, cudaStream_t s) {
  if (g.n == 0) return GF_OK;
  FwdArgs<T> a = a0;
  const FastShape fs = fast_shape(a.H, a.D, sizeof(T));
  const bool al = aligned16(a.V) && aligned16(a.O) &&
                  (variant == GF_ADD || (aligned16(a.Q) && aligned16(a.K)));
  if (fs.ok && al) {
    a.GD = fs.gd;
    const int warp_rows = g.n - a.n_cta;
    const int blocks = a.n_cta + (warp_rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    switch (fs.lpe * 8 + fs.cpl) {
      case 1 * 8 + 1: return launch_fast_fwd<T, 1, 1>(a, variant, blocks, s);
      case 2 * 8 + 1: return launch_fast_fwd<T, 2, 1>(a, variant, blocks, s);
      case 4 * 8 + 1: return launch_fast_fwd<T, 4, 1>(a, variant, blocks, s);
      case 8 * 8 + 1: return launch_fast_fwd<T, 8, 1>(a, variant, blocks, s);
      case 16 * 8 + 1: return launch_fast_fwd<T, 16, 1>(a, variant, blocks, s);
      case 32 * 8 + 1: return launch_fast_fwd<T, 32, 1>(a, variant, blocks, s);
      case 32 * 8 + 2: return launch_fast_fwd<T, 32, 2>(a, variant, blocks, s);
      case 32 * 8 + 4: return launch_fast_fwd<T, 32, 4>(a, variant, blocks, s);
      default: break;
    }
  }
  if (a.H > 32) {
    set_error("gf_attn_fwd: heads > 32 need a head shape that tiles into 16-byte chunks");
    return GF_ERR_UNSUPPORTED;
  }
  const size_t smem = static_cast<size_t>(kGenericWarps) * (2 * a.F + 64) * sizeof(T);
  if (smem > 200 * 1024) {
    set_error("gf_attn_fwd: feature width too large for the generic path");
    return GF_ERR_UNSUPPORTED;
  }
  const int blocks = (g.n + kGenericWarps - 1) / kGenericWarps;
  if (variant == GF_DOT) {
    if (smem > 48 * 1024)
      GF_CHECK_CUDA(cudaFuncSetAttribute(fwd_generic<T, GF_DOT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    fwd_generic<T, GF_DOT><<<blocks, 32 * kGenericWarps, smem, s>>>(a);
  } else {
    if (smem > 48 * 1024)
      GF_CHECK_CUDA(cudaFuncSetAttribute(fwd_generic<T, GF_ADD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    fwd_generic<T, GF_ADD><<<blocks, 32 * kGenericWarps, smem, s>>>(a);
  }
  GF_CHECK_LAUNCH("fwd_generic");
  return GF_OK;
}

template <typename T>
int launch_materialize_p(const DevGraph& g, const FwdArgs<T>& a, int variant, T* P,
                         cudaStream_t s) {
  if (g.n == 0 || g.e == 0) return GF_OK;
  if (a.H > 32) {
    set_error("gf_attn_fwd: P materialisation supports heads <= 32");
    return GF_ERR_UNSUPPORTED;
  }
  const int blocks = (g.n + kGenericWarps - 1) / kGenericWarps;
  if (variant == GF_DOT)
    materialize_p<T, GF_DOT><<<blocks, 32 * kGenericWarps, 0, s>>>(a, P);
  else
    materialize_p<T, GF_ADD><<<blocks, 32 * kGenericWarps, 0, s>>>(a, P);
  GF_CHECK_LAUNCH("materialize_p");
  return GF_OK;
}

template int launch_fwd<float>(const DevGraph&, const FwdArgs<float>&, int, cudaStream_t);
template int launch_fwd<double>(const DevGraph&, const FwdArgs<double>&, int, cudaStream_t);
template int launch_materialize_p<float>(const DevGraph&, const FwdArgs<float>&, int, float*,
                                         cudaStream_t);
template int launch_materialize_p<double>(const DevGraph&, const FwdArgs<double>&, int, double*,
                                          cudaStream_t);

}  // namespace gfb

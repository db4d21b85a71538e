// Recompute backward of the fused AT-GNN layer for sm_100a.  Replaces the
// reference's serial backward_values (autograd.hpp:158-170) =
// spmm_backward (33-58) -> softmax_backward (62-73) -> sddmm_backward
// (102-154), and the AGNN chain l2_normalize_backward (76-95).
//
// No E x H tensor is stored or read: attention is recomputed per edge from
// the forward statistics (row max, log-sum; N x H x 2), and the softmax-Jacobian row term
// sum_row P*dP is the per-destination scalar delta = <dO[v], O[v]> (exact
// identity, since O[v] = sum P V).  Two owner-computes passes, no atomics:
//
//   pass A (CSR rows, destination-owned), per in-edge u -> v:
//       s = score(u, v); p = exp((s - m[v]) - logl[v]); dP = <dO[v], V[u]>;
//       dS = p (dP - delta[v])
//       dot: dK[v] += scale dS Qhat[u]       add: der[v] += dS lrelu'(pre)
//     also writes delta[v] for pass B.
//   pass B (CSC columns, source-owned), per out-edge u -> v:
//       same p, dS from (m[v], logl[v], delta[v], K[v] | er[v], dO[v])
//       dV[u] += p dO[v];  dot: dQ[u] += scale dS Khat[v]
//                          add: del[u] += dS lrelu'(pre)
// AGNN's L2 Jacobian is applied in each pass's epilogue on the owned row.
// Scheduling mirrors the forward: degree-descending order, CTA rows for
// degree >= cta_threshold (8 balanced slices merged in shared memory in a
// fixed order), warp rows otherwise.
#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace gfb {

namespace {

// L2 backward on one owned row (autograd.hpp:76-95): g holds dXhat, x the raw
// row; the head norm is reduced over the head's lanes.  Returns dX in g.
template <typename T, int LPE, int CPL, int CW>
__device__ __forceinline__ void l2_backward_rows(T (&g)[CPL][CW], const T (&x)[CPL][CW], int gd) {
  const T eps = T(1e-12);
  T sq[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    T s = T(0);
#pragma unroll
    for (int i = 0; i < CW; ++i) s += x[k][i] * x[k][i];
    sq[k] = s;
  }
  head_sum<LPE, CPL>(sq, gd);
  T nrm[CPL], dot[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    nrm[k] = sqrt(sq[k]);
    T d = T(0);
    if (nrm[k] > eps) {
#pragma unroll
      for (int i = 0; i < CW; ++i) d += x[k][i] / nrm[k] * g[k][i];
    }
    dot[k] = d;
  }
  head_sum<LPE, CPL>(dot, gd);
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    if (nrm[k] <= eps) {
#pragma unroll
      for (int i = 0; i < CW; ++i) g[k][i] = g[k][i] / eps;
    } else {
#pragma unroll
      for (int i = 0; i < CW; ++i) g[k][i] = (g[k][i] - x[k][i] / nrm[k] * dot[k]) / nrm[k];
    }
  }
}

// Sum-merge of per-warp partials through shared memory (fixed warp order).
// After the call, every lane of warp 0 holds the CTA total; other warps
// return false.
template <typename T, int LPE, int NV>
__device__ __forceinline__ bool cta_sum(T (&x)[NV], int warp, int c, int sub) {
  __shared__ T sm[kWarpsPerBlock][LPE][NV];
  if (sub == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[warp][c][j] = x[j];
  }
  __syncthreads();
  if (warp != 0) return false;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    T s = sm[0][c][j];
    for (int w = 1; w < kWarpsPerBlock; ++w) s += sm[w][c][j];
    x[j] = s;
  }
  return true;
}

// ------------------------------------------------------------ pass A ------
template <typename T, int LPE, int CPL, int VAR>
__global__ void __launch_bounds__(256) bwd_rows_fast(const BwdArgs<T> a) {
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
  const size_t vrow = static_cast<size_t>(v) * a.F;

  T dov[CPL][CW], delta[CPL], mv[CPL], llv[CPL];
  {
    T ov[CPL][CW];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      ld_chunk(a.dO + vrow + off[k], dov[k]);
      ld_chunk(a.O + vrow + off[k], ov[k]);
      T s = T(0);
#pragma unroll
      for (int i = 0; i < CW; ++i) s += dov[k][i] * ov[k][i];
      delta[k] = s;
      ld_stat(a.stats, static_cast<size_t>(v) * a.H + head[k], mv[k], llv[k]);
    }
    head_sum<LPE, CPL>(delta, a.GD);
  }
  T kv[CPL][CW], erv[CPL], rk[CPL];
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) ld_chunk(a.K + vrow + off[k], kv[k]);
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

  // Accumulators: dot -> dKhat chunks; add -> der per chunk's head.
  T acc[CPL * (VAR == GF_DOT ? CW : 1)];
#pragma unroll
  for (int j = 0; j < CPL * (VAR == GF_DOT ? CW : 1); ++j) acc[j] = T(0);

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
      T vv[U][CPL][CW], qv[U][CPL][CW], elv[U][CPL];
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
        T s[CPL], dp[CPL], rq[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          T d = T(0);
#pragma unroll
          for (int i = 0; i < CW; ++i) d += dov[k][i] * vv[t][k][i];
          dp[k] = d;
        }
        head_sum<LPE, CPL>(dp, a.GD);
        if constexpr (VAR == GF_DOT) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            T d = T(0), qq = T(0);
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              d += qv[t][k][i] * kv[k][i];
              qq += qv[t][k][i] * qv[t][k][i];
            }
            s[k] = d;
            rq[k] = qq;
          }
          head_sum<LPE, CPL>(s, a.GD);
          if (a.l2) {
            head_sum<LPE, CPL>(rq, a.GD);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              rq[k] = inv_norm(rq[k]);
              s[k] = a.scale * s[k] * (rq[k] * rk[k]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              rq[k] = T(1);
              s[k] = a.scale * s[k];
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < CPL; ++k) s[k] = lrelu(elv[t][k] + erv[k], a.slope);
        }
        if (ok[t]) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const T p = prob(s[k], mv[k], llv[k]);
            const T ds = p * (dp[k] - delta[k]);
            if constexpr (VAR == GF_DOT) {
              const T w = a.scale * ds * rq[k];
#pragma unroll
              for (int i = 0; i < CW; ++i) acc[k * CW + i] += w * qv[t][k][i];
            } else {
              acc[k] += ds * lrelu_grad(elv[t][k] + erv[k], a.slope);
            }
          }
        }
      }
    }
  }

  constexpr int NA = CPL * (VAR == GF_DOT ? CW : 1);
#pragma unroll
  for (int o = LPE; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], o);
  }
  if (cta && !cta_sum<T, LPE, NA>(acc, warp, c, sub)) return;

  if constexpr (VAR == GF_DOT) {
    T g[CPL][CW];
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
      for (int i = 0; i < CW; ++i) g[k][i] = acc[k * CW + i];
    if (a.l2) l2_backward_rows<T, LPE, CPL, CW>(g, kv, a.GD);
    if (sub == 0) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) st_chunk(a.dK + vrow + off[k], g[k]);
    }
  }
  if (sub == 0) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      if ((c + k * LPE) % a.GD == 0) {
        const size_t hi = static_cast<size_t>(v) * a.H + head[k];
        a.delta[hi] = delta[k];
        if constexpr (VAR == GF_ADD) a.dK[hi] = acc[k];
      }
    }
  }
}

// ------------------------------------------------------------ pass B ------
template <typename T, int LPE, int CPL, int VAR>
__global__ void __launch_bounds__(256) bwd_cols_fast(const BwdArgs<T> a) {
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
  const int u = __ldg(a.order + slot);
  int sb = __ldg(a.ptr + u), se = __ldg(a.ptr + u + 1);
  if (cta) split_range(sb, se, kWarpsPerBlock, warp, sb, se);

  int off[CPL], head[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const int ch = c + k * LPE;
    off[k] = ch * CW;
    head[k] = ch / a.GD;
  }
  const size_t urow = static_cast<size_t>(u) * a.F;

  // Source-side operands owned by this column.
  T vu[CPL][CW], qu[CPL][CW], elu[CPL], rq[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) ld_chunk(a.V + urow + off[k], vu[k]);
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) ld_chunk(a.Q + urow + off[k], qu[k]);
    if (a.l2) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        T s = T(0);
#pragma unroll
        for (int i = 0; i < CW; ++i) s += qu[k][i] * qu[k][i];
        rq[k] = s;
      }
      head_sum<LPE, CPL>(rq, a.GD);
#pragma unroll
      for (int k = 0; k < CPL; ++k) rq[k] = inv_norm(rq[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < CPL; ++k) elu[k] = __ldg(a.Q + static_cast<size_t>(u) * a.H + head[k]);
  }

  T dv[CPL][CW];
  T acc[CPL * (VAR == GF_DOT ? CW : 1)];
#pragma unroll
  for (int k = 0; k < CPL; ++k)
#pragma unroll
    for (int i = 0; i < CW; ++i) dv[k][i] = T(0);
#pragma unroll
  for (int j = 0; j < CPL * (VAR == GF_DOT ? CW : 1); ++j) acc[j] = T(0);

  for (int base = sb; base < se; base += 32) {
    const int cnt = min(32, se - base);
    const int myv = lane < cnt ? __ldg(a.idx + base + lane) : 0;
#pragma unroll 1
    for (int j0 = 0; j0 < cnt; j0 += EPW * U) {
      int vv[U];
      bool ok[U];
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const int j = j0 + t * EPW + sub;
        ok[t] = j < cnt;
        vv[t] = __shfl_sync(kFull, myv, j & 31);
      }
      T dov[U][CPL][CW], kv[U][CPL][CW], mv[U][CPL], llv[U][CPL], dlt[U][CPL], erv[U][CPL];
#pragma unroll
      for (int t = 0; t < U; ++t) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const size_t vrow = static_cast<size_t>(vv[t]) * a.F;
          const size_t hi = static_cast<size_t>(vv[t]) * a.H + head[k];
          if (ok[t]) {
            ld_chunk(a.dO + vrow + off[k], dov[t][k]);
            if constexpr (VAR == GF_DOT)
              ld_chunk(a.K + vrow + off[k], kv[t][k]);
            else
              erv[t][k] = __ldg(a.K + hi);
            ld_stat(a.stats, hi, mv[t][k], llv[t][k]);
            dlt[t][k] = __ldg(a.delta + hi);
          } else {
#pragma unroll
            for (int i = 0; i < CW; ++i) dov[t][k][i] = T(0), kv[t][k][i] = T(0);
            erv[t][k] = T(0);
            mv[t][k] = T(0);
            llv[t][k] = T(0);
            dlt[t][k] = T(0);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < U; ++t) {
        T s[CPL], dp[CPL], rk[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          T d = T(0);
#pragma unroll
          for (int i = 0; i < CW; ++i) d += dov[t][k][i] * vu[k][i];
          dp[k] = d;
        }
        head_sum<LPE, CPL>(dp, a.GD);
        if constexpr (VAR == GF_DOT) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            T d = T(0), kk = T(0);
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              d += qu[k][i] * kv[t][k][i];
              kk += kv[t][k][i] * kv[t][k][i];
            }
            s[k] = d;
            rk[k] = kk;
          }
          head_sum<LPE, CPL>(s, a.GD);
          if (a.l2) {
            head_sum<LPE, CPL>(rk, a.GD);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              rk[k] = inv_norm(rk[k]);
              s[k] = a.scale * s[k] * (rq[k] * rk[k]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              rk[k] = T(1);
              s[k] = a.scale * s[k];
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < CPL; ++k) s[k] = lrelu(elu[k] + erv[t][k], a.slope);
        }
        if (ok[t]) {
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const T p = prob(s[k], mv[t][k], llv[t][k]);
            const T ds = p * (dp[k] - dlt[t][k]);
#pragma unroll
            for (int i = 0; i < CW; ++i) dv[k][i] += p * dov[t][k][i];
            if constexpr (VAR == GF_DOT) {
              const T w = a.scale * ds * rk[k];
#pragma unroll
              for (int i = 0; i < CW; ++i) acc[k * CW + i] += w * kv[t][k][i];
            } else {
              acc[k] += ds * lrelu_grad(elu[k] + erv[t][k], a.slope);
            }
          }
        }
      }
    }
  }

  constexpr int NA = CPL * (VAR == GF_DOT ? CW : 1);
  constexpr int NT = CPL * CW + NA;
  T all[NT];
#pragma unroll
  for (int k = 0; k < CPL; ++k)
#pragma unroll
    for (int i = 0; i < CW; ++i) all[k * CW + i] = dv[k][i];
#pragma unroll
  for (int j = 0; j < NA; ++j) all[CPL * CW + j] = acc[j];
#pragma unroll
  for (int o = LPE; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < NT; ++j) all[j] += __shfl_xor_sync(kFull, all[j], o);
  }
  if (cta && !cta_sum<T, LPE, NT>(all, warp, c, sub)) return;

  T g[CPL][CW];
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
      for (int i = 0; i < CW; ++i) g[k][i] = all[CPL * CW + k * CW + i];
    if (a.l2) l2_backward_rows<T, LPE, CPL, CW>(g, qu, a.GD);
  }
  if (sub == 0) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      T o[CW];
#pragma unroll
      for (int i = 0; i < CW; ++i) o[i] = all[k * CW + i];
      st_chunk(a.dV + urow + off[k], o);
      if constexpr (VAR == GF_DOT) {
        st_chunk(a.dQ + urow + off[k], g[k]);
      } else {
        if ((c + k * LPE) % a.GD == 0)
          a.dQ[static_cast<size_t>(u) * a.H + head[k]] = all[CPL * CW + k];
      }
    }
  }
}

// ----------------------------------------------------------- generic path --
// Serial-per-head versions for shapes that do not tile into 16-byte chunks.
template <typename T, int VAR>
__global__ void __launch_bounds__(128) bwd_rows_generic(const BwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * kGenericWarps + warp;
  if (slot >= a.n) return;
  T* ws = reinterpret_cast<T*>(smraw) + static_cast<size_t>(warp) * (3 * a.F + 32);
  T* dos = ws;          // dO[v]
  T* kvs = ws + a.F;    // K[v]
  T* gk = ws + 2 * a.F; // dKhat[v]
  T* wh = ws + 3 * a.F; // per-head edge weight
  const int v = __ldg(a.order + slot);
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  const size_t vrow = static_cast<size_t>(v) * a.F;
  for (int f = lane; f < a.F; f += 32) {
    dos[f] = __ldg(a.dO + vrow + f);
    if constexpr (VAR == GF_DOT) kvs[f] = __ldg(a.K + vrow + f);
    gk[f] = T(0);
  }
  __syncwarp();
  T erh, rkh;
  generic_row_setup<T, VAR>(a, v, lane, VAR == GF_DOT ? kvs : nullptr, erh, rkh);
  T dlt = T(0), mh = T(0), llh = T(0), gr = T(0);
  if (lane < a.H) {
    for (int j = 0; j < a.D; ++j) dlt += dos[lane * a.D + j] * __ldg(a.O + vrow + lane * a.D + j);
    a.delta[static_cast<size_t>(v) * a.H + lane] = dlt;
    ld_stat(a.stats, static_cast<size_t>(v) * a.H + lane, mh, llh);
  }
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    if (lane < a.H) {
      T rq = T(1), pre = T(0);
      const T s = generic_score<T, VAR>(a, u, v, lane, kvs, erh, rkh, &rq, &pre);
      const T p = prob(s, mh, llh);
      T dp = T(0);
      for (int j = 0; j < a.D; ++j)
        dp += dos[lane * a.D + j] * __ldg(a.V + static_cast<size_t>(u) * a.F + lane * a.D + j);
      const T ds = p * (dp - dlt);
      if constexpr (VAR == GF_DOT)
        wh[lane] = a.scale * ds * rq;
      else
        gr += ds * lrelu_grad(pre, a.slope);
    }
    if constexpr (VAR == GF_DOT) {
      __syncwarp();
      for (int f = lane; f < a.F; f += 32)
        gk[f] += wh[f / a.D] * __ldg(a.Q + static_cast<size_t>(u) * a.F + f);
      __syncwarp();
    }
  }
  if constexpr (VAR == GF_ADD) {
    if (lane < a.H) a.dK[static_cast<size_t>(v) * a.H + lane] = gr;
  } else {
    __syncwarp();
    if (a.l2) {
      if (lane < a.H) {
        const T eps = T(1e-12);
        const T* x = kvs + lane * a.D;
        T* g = gk + lane * a.D;
        T sq = T(0);
        for (int j = 0; j < a.D; ++j) sq += x[j] * x[j];
        const T nrm = sqrt(sq);
        if (nrm <= eps) {
          for (int j = 0; j < a.D; ++j) g[j] = g[j] / eps;
        } else {
          T dot = T(0);
          for (int j = 0; j < a.D; ++j) dot += x[j] / nrm * g[j];
          for (int j = 0; j < a.D; ++j) g[j] = (g[j] - x[j] / nrm * dot) / nrm;
        }
      }
      __syncwarp();
    }
    for (int f = lane; f < a.F; f += 32) a.dK[vrow + f] = gk[f];
  }
}

template <typename T, int VAR>
__global__ void __launch_bounds__(128) bwd_cols_generic(const BwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * kGenericWarps + warp;
  if (slot >= a.n) return;
  T* ws = reinterpret_cast<T*>(smraw) + static_cast<size_t>(warp) * (4 * a.F + 64);
  T* vus = ws;            // V[u]
  T* qus = ws + a.F;      // Q[u]
  T* dva = ws + 2 * a.F;  // dV[u]
  T* gq = ws + 3 * a.F;   // dQhat[u]
  T* ph = ws + 4 * a.F;   // 32
  T* wh = ph + 32;        // 32
  const int u = __ldg(a.order + slot);
  const int sb = __ldg(a.ptr + u), se = __ldg(a.ptr + u + 1);
  const size_t urow = static_cast<size_t>(u) * a.F;
  for (int f = lane; f < a.F; f += 32) {
    vus[f] = __ldg(a.V + urow + f);
    if constexpr (VAR == GF_DOT) qus[f] = __ldg(a.Q + urow + f);
    dva[f] = T(0);
    gq[f] = T(0);
  }
  __syncwarp();
  T elh = T(0), rqh = T(1), gl = T(0);
  if (lane < a.H) {
    if constexpr (VAR == GF_ADD) {
      elh = __ldg(a.Q + static_cast<size_t>(u) * a.H + lane);
    } else if (a.l2) {
      T s = T(0);
      for (int j = 0; j < a.D; ++j) s += qus[lane * a.D + j] * qus[lane * a.D + j];
      rqh = inv_norm(s);
    }
  }
  for (int i = sb; i < se; ++i) {
    const int v = __ldg(a.idx + i);
    const size_t vrow = static_cast<size_t>(v) * a.F;
    if (lane < a.H) {
      const size_t hi = static_cast<size_t>(v) * a.H + lane;
      T s, pre = T(0), rk = T(1);
      if constexpr (VAR == GF_DOT) {
        T d = T(0), kk = T(0);
        for (int j = 0; j < a.D; ++j) {
          const T x = __ldg(a.K + vrow + lane * a.D + j);
          d += qus[lane * a.D + j] * x;
          kk += x * x;
        }
        if (a.l2) {
          rk = inv_norm(kk);
          s = a.scale * d * (rqh * rk);
        } else {
          s = a.scale * d;
        }
      } else {
        pre = elh + __ldg(a.K + hi);
        s = lrelu(pre, a.slope);
      }
      T mh, llh;
      ld_stat(a.stats, hi, mh, llh);
      const T p = prob(s, mh, llh);
      T dp = T(0);
      for (int j = 0; j < a.D; ++j) dp += __ldg(a.dO + vrow + lane * a.D + j) * vus[lane * a.D + j];
      const T ds = p * (dp - __ldg(a.delta + hi));
      ph[lane] = p;
      if constexpr (VAR == GF_DOT)
        wh[lane] = a.scale * ds * rk;
      else
        gl += ds * lrelu_grad(pre, a.slope);
    }
    __syncwarp();
    for (int f = lane; f < a.F; f += 32) {
      dva[f] += ph[f / a.D] * __ldg(a.dO + vrow + f);
      if constexpr (VAR == GF_DOT) gq[f] += wh[f / a.D] * __ldg(a.K + vrow + f);
    }
    __syncwarp();
  }
  for (int f = lane; f < a.F; f += 32) a.dV[urow + f] = dva[f];
  if constexpr (VAR == GF_ADD) {
    if (lane < a.H) a.dQ[static_cast<size_t>(u) * a.H + lane] = gl;
  } else {
    if (a.l2) {
      if (lane < a.H) {
        const T eps = T(1e-12);
        const T* x = qus + lane * a.D;
        T* g = gq + lane * a.D;
        T sq = T(0);
        for (int j = 0; j < a.D; ++j) sq += x[j] * x[j];
        const T nrm = sqrt(sq);
        if (nrm <= eps) {
          for (int j = 0; j < a.D; ++j) g[j] = g[j] / eps;
        } else {
          T dot = T(0);
          for (int j = 0; j < a.D; ++j) dot += x[j] / nrm * g[j];
          for (int j = 0; j < a.D; ++j) g[j] = (g[j] - x[j] / nrm * dot) / nrm;
        }
      }
      __syncwarp();
    }
    for (int f = lane; f < a.F; f += 32) a.dQ[urow + f] = gq[f];
  }
}

template <typename T, int LPE, int CPL>
int launch_fast_bwd(const BwdArgs<T>& ra, const BwdArgs<T>& ca, int variant, int rblocks,
                    int cblocks, cudaStream_t s) {
  if (variant == GF_DOT) {
    if (rblocks) bwd_rows_fast<T, LPE, CPL, GF_DOT><<<rblocks, 256, 0, s>>>(ra);
    GF_CHECK_LAUNCH("bwd_rows_fast");
    if (cblocks) bwd_cols_fast<T, LPE, CPL, GF_DOT><<<cblocks, 256, 0, s>>>(ca);
    GF_CHECK_LAUNCH("bwd_cols_fast");
  } else {
    if (rblocks) bwd_rows_fast<T, LPE, CPL, GF_ADD><<<rblocks, 256, 0, s>>>(ra);
    GF_CHECK_LAUNCH("bwd_rows_fast");
    if (cblocks) bwd_cols_fast<T, LPE, CPL, GF_ADD><<<cblocks, 256, 0, s>>>(ca);
    GF_CHECK_LAUNCH("bwd_cols_fast");
  }
  return GF_OK;
}

template <typename K>
int set_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024)
    GF_CHECK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  return GF_OK;
}

}  // namespace

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
int launch_bwd(const DevGraph& g, BwdArgs<T> a, int variant, int passes, cudaStream_t s) {
  if (g.n == 0) return GF_OK;
  BwdArgs<T> ra = a, ca = a;
  ra.ptr = g.row_ptr, ra.idx = g.col, ra.order = g.row_order, ra.n_cta = g.n_cta_rows;
  ca.ptr = g.csc_ptr, ca.idx = g.csc_row, ca.order = g.col_order, ca.n_cta = g.n_cta_cols;
  const bool do_a = passes & 1, do_b = passes & 2;
  const bool dot = variant == GF_DOT;
  // Each pass picks the fast path independently (both paths write the same
  // delta), so a misaligned operand of one pass never affects the other.
  const FastShape fs = fast_shape(a.H, a.D, sizeof(T));
  const bool fast_a = fs.ok && aligned16(a.V) && aligned16(a.O) && aligned16(a.dO) &&
                      (!dot || (aligned16(a.Q) && aligned16(a.K) && aligned16(a.dK)));
  const bool fast_b = fs.ok && aligned16(a.V) && aligned16(a.dO) && aligned16(a.dV) &&
                      (!dot || (aligned16(a.Q) && aligned16(a.K) && aligned16(a.dQ)));
  ra.GD = ca.GD = fs.ok ? fs.gd : 1;
  const int rb = (do_a && fast_a) ? ra.n_cta + (g.n - ra.n_cta + kWarpsPerBlock - 1) / kWarpsPerBlock : 0;
  const int cb = (do_b && fast_b) ? ca.n_cta + (g.n - ca.n_cta + kWarpsPerBlock - 1) / kWarpsPerBlock : 0;
  if (rb || cb) {
    int rc = GF_OK;
    switch (fs.lpe * 8 + fs.cpl) {
      case 1 * 8 + 1: rc = launch_fast_bwd<T, 1, 1>(ra, ca, variant, rb, cb, s); break;
      case 2 * 8 + 1: rc = launch_fast_bwd<T, 2, 1>(ra, ca, variant, rb, cb, s); break;
      case 4 * 8 + 1: rc = launch_fast_bwd<T, 4, 1>(ra, ca, variant, rb, cb, s); break;
      case 8 * 8 + 1: rc = launch_fast_bwd<T, 8, 1>(ra, ca, variant, rb, cb, s); break;
      case 16 * 8 + 1: rc = launch_fast_bwd<T, 16, 1>(ra, ca, variant, rb, cb, s); break;
      case 32 * 8 + 1: rc = launch_fast_bwd<T, 32, 1>(ra, ca, variant, rb, cb, s); break;
      case 32 * 8 + 2: rc = launch_fast_bwd<T, 32, 2>(ra, ca, variant, rb, cb, s); break;
      case 32 * 8 + 4: rc = launch_fast_bwd<T, 32, 4>(ra, ca, variant, rb, cb, s); break;
      default: set_error("gf_attn_bwd: internal fast-shape dispatch"); return GF_ERR_CUDA;
    }
    if (rc) return rc;
  }
  const bool gen_a = do_a && !fast_a, gen_b = do_b && !fast_b;
  if (!gen_a && !gen_b) return GF_OK;
  if (a.H > 32) {
    set_error("gf_attn_bwd: heads > 32 need a head shape that tiles into 16-byte chunks");
    return GF_ERR_UNSUPPORTED;
  }
  const size_t sa = static_cast<size_t>(kGenericWarps) * (3 * a.F + 32) * sizeof(T);
  const size_t sb = static_cast<size_t>(kGenericWarps) * (4 * a.F + 64) * sizeof(T);
  if (sb > 200 * 1024) {
    set_error("gf_attn_bwd: feature width too large for the generic path");
    return GF_ERR_UNSUPPORTED;
  }
  const int blocks = (g.n + kGenericWarps - 1) / kGenericWarps;
  int rc;
  if (dot) {
    if (gen_a) {
      if ((rc = set_smem(bwd_rows_generic<T, GF_DOT>, sa))) return rc;
      bwd_rows_generic<T, GF_DOT><<<blocks, 32 * kGenericWarps, sa, s>>>(ra);
      GF_CHECK_LAUNCH("bwd_rows_generic");
    }
    if (gen_b) {
      if ((rc = set_smem(bwd_cols_generic<T, GF_DOT>, sb))) return rc;
      bwd_cols_generic<T, GF_DOT><<<blocks, 32 * kGenericWarps, sb, s>>>(ca);
      GF_CHECK_LAUNCH("bwd_cols_generic");
    }
  } else {
    if (gen_a) {
      if ((rc = set_smem(bwd_rows_generic<T, GF_ADD>, sa))) return rc;
      bwd_rows_generic<T, GF_ADD><<<blocks, 32 * kGenericWarps, sa, s>>>(ra);
      GF_CHECK_LAUNCH("bwd_rows_generic");
    }
    if (gen_b) {
      if ((rc = set_smem(bwd_cols_generic<T, GF_ADD>, sb))) return rc;
      bwd_cols_generic<T, GF_ADD><<<blocks, 32 * kGenericWarps, sb, s>>>(ca);
      GF_CHECK_LAUNCH("bwd_cols_generic");
    }
  }
  return GF_OK;
}

template int launch_bwd<float>(const DevGraph&, BwdArgs<float>, int, int, cudaStream_t);
template int launch_bwd<double>(const DevGraph&, BwdArgs<double>, int, int, cudaStream_t);

}  // namespace gfb

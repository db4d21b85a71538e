#pragma once
// (Included by gf_attn_bwd_f32.cu / gf_attn_bwd_f64.cu, one translation unit
// per element type, compiled in parallel.)
//
// Recompute backward of the fused AT-GNN layer for sm_100a.  Replaces the
// reference's serial backward_values (autograd.hpp:158-170) =
// spmm_backward (33-58) -> softmax_backward (62-73) -> sddmm_backward
// (102-154), and the AGNN chain l2_normalize_backward (76-95).
//
// No E x H tensor is stored or read: attention is recomputed per edge from
// the forward's per-(row, head) records {m, log2 l, aux, delta}, and the
// softmax-Jacobian row term sum_row P*dP is the per-destination scalar
// delta = <dO[v], O[v]> (exact identity, since O[v] = sum P V).  Two
// owner-computes passes, no atomics:
//
//   pass A (CSR rows, destination-owned), per in-edge u -> v:
//       s = score(u, v); p = exp(s - m[v]) / l[v]; dP = <dO[v], V[u]>;
//       dS = p (dP - delta[v])
//       dot: dK[v] += scale dS Qhat[u]       add: der[v] += dS lrelu'(pre)
//     and writes delta[v] into the record for pass B.
//   pass B (CSC columns, source-owned), per out-edge u -> v:
//       one 16 B record gather gives (m, log2 l, er|1/||K||, delta) of v;
//       dV[u] += p dO[v];  dot: dQ[u] += scale dS Khat[v]
//                          add: del[u] += dS lrelu'(pre)
// AGNN's L2 Jacobian is applied in each pass's epilogue on the owned row.
// Scheduling and lane mapping mirror the forward (gf_attn_fwd.cuh).
#include <type_traits>

#include "gf_device.cuh"
#include "gf_internal.cuh"

#ifndef GF_FULL_CHUNK_A
#define GF_FULL_CHUNK_A 1
#endif
#ifndef GF_FULL_CHUNK_B
#define GF_FULL_CHUNK_B 1
#endif

#ifndef GF_FULL_STEPS
#define GF_FULL_STEPS 0
#endif

namespace gfb {

// Per-edge dot products of the backward passes (dP = <dO, V>, the dot
// scores): paired FFMA2 (half the dependent FMA chain) or the sequential
// order.  Measured per pass (profiles/r2/ab_r2_policy_param.txt): pairs help
// pass B (-1.5 %) and the table-form pass A (-2 %), but cost the GAT
// layer-form pass A 20 % (its 64-register budget), which keeps the sequence.
#ifndef GF_BWD_LPH1
#define GF_BWD_LPH1 1  // pass A, GAT layer-form warp rows with LPH = 1 at compile time
#endif
#ifndef GF_BWDC_LPH1
#define GF_BWDC_LPH1 1  // the same for pass B warp columns (C4 pass B -2.5 %)
#endif
#ifndef GF_BWD_LPH1_TABLE
#define GF_BWD_LPH1_TABLE 1  // both passes' LPH = 1 copies for the el / er table form too (table-form step +2 %)
#endif
#ifndef GF_BWD_DOT2
#define GF_BWD_DOT2 1
#endif
template <bool PAIRED, typename T, int N>
__device__ __forceinline__ T bdot(const T (&x)[N], const T (&y)[N]) {
  if constexpr (PAIRED && GF_BWD_DOT2) {
    return dot_n(x, y);
  } else {
    T s = T(0);
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i] * y[i];
    return s;
  }
}

namespace {

// L2 backward of one owned head row (autograd.hpp:76-95): g holds dXhat, x
// the raw row; norms reduced over the LPH lanes of the head.
template <typename T, int NE>
__device__ __forceinline__ void l2_backward_row(T (&g)[NE], const T (&x)[NE], int lph) {
  const T eps = T(1e-12);
  T sq = T(0);
#pragma unroll
  for (int i = 0; i < NE; ++i) sq += x[i] * x[i];
  const T nrm = sqrt(head_sum(sq, lph));
  T d = T(0);
  if (nrm > eps) {
#pragma unroll
    for (int i = 0; i < NE; ++i) d += x[i] / nrm * g[i];
  }
  const T dot = head_sum(d, lph);
  if (nrm <= eps) {
#pragma unroll
    for (int i = 0; i < NE; ++i) g[i] = g[i] / eps;
  } else {
#pragma unroll
    for (int i = 0; i < NE; ++i) g[i] = (g[i] - x[i] / nrm * dot) / nrm;
  }
}

// Sum-merge of per-warp partials through shared memory (fixed warp order).
// Every lane of warp 0 ends with the CTA total; other warps return false.
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

template <typename T, int LPE, int NV>
__device__ __forceinline__ void warp_sum(T (&x)[NV]) {
#pragma unroll
  for (int o = LPE; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < NV; ++j) x[j] += __shfl_xor_sync(kFull, x[j], o);
  }
}

// ------------------------------------------------------------ pass A ------
template <typename T, int CB, int LPE, int CPL, int VAR, bool PK, int LPHC = 0>
__device__ __forceinline__ void bwd_row(const BwdArgs<T>& a, const int lane, const int warp,
                                        const bool cta, const int slot, const bool live,
                                        const int nrows, const int4 ct) {
  const int lph = LPHC ? LPHC : a.LPH;  // compile-time 1 for GAT layer-form warp rows (as fwd_row)
  constexpr int CW = Chunk<T, CB>::W;
  constexpr int NE = CPL * CW;
  constexpr int EPW = 32 / LPE;
  constexpr int U = CPL == 1 ? (VAR == GF_ADDV ? GF_U_ROWS_V : VAR == GF_DOT ? GF_U_DOT1 : GF_U_ROWS)
                             : (PK ? GF_U2_PK : GF_U2);
  constexpr int NA = VAR == GF_DOT ? NE : 1;
  constexpr bool pk = PK;  // packed row: this LPE-lane group owns the row
  const int c = lane % LPE, sub = lane / LPE;
  // nrows consecutive warp rows, software-pipelined like fwd_row (gf_attn_fwd.cuh)
  const int4 zero4 = make_int4(0, 0, 0, 0);
  constexpr bool PKPRE = PK && LPE >= kSmallDegree;  // packed rows: ids loaded up front
  int4 rs;
  if constexpr (GF_SCHED16_ROWS || PK) {
    rs = live ? ld_sched(a.sched + slot) : zero4;
  } else {
    const int v0 = live ? __ldg(a.order + slot) : 0;
    rs = live ? make_int4(v0, __ldg(a.ptr + v0), __ldg(a.ptr + v0 + 1), 0) : zero4;
  }
  int4 rsn = nrows > 1 ? ld_sched(a.sched + slot + 1) : zero4;
  int nxt = 0;
  for (int r = 0; r < nrows; ++r) {
  const int4 rsnn = r + 2 < nrows ? ld_sched(a.sched + slot + r + 2) : zero4;
  const int v = rs.x;
  int eb = rs.y, ee = rs.z;
  if (cta) {
    if (ct.z > 1) split_range(eb, ee, ct.z, ct.y, eb, ee);  // this CTA's slice of a split row
    split_range(eb, ee, kWarpsPerBlock, warp, eb, ee);
  }
  if (r == 0 && !pk) nxt = eb + lane < ee ? ld_idx(a.idx + eb + lane) : 0;
  if constexpr (PKPRE) nxt = c < ee - eb ? ld_idx(a.idx + eb + c) : 0;

  const int h = c / lph;
  const int off = h * a.D + (c % lph) * NE;
  const size_t vrow = static_cast<size_t>(v) * a.F + off;
  const size_t ri = static_cast<size_t>(v) * a.H + h;
  const T* __restrict__ Vb = a.V + off;
  const T* __restrict__ Qb = a.Q + (VAR == GF_DOT ? off : h);
  const int qs = VAR == GF_DOT ? a.F : a.H;
  const uint32_t fb = a.F * sizeof(T), qb = qs * sizeof(T);  // row strides in bytes
  const uint64_t pol = GF_POL_PARAM_BWD ? a.pol : pol_keep();
  T al[NE];  // GF_ADDV: el = <V[u], a_l> from the gathered V row
  if constexpr (VAR == GF_ADDV) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.Q + off + k * CW, *reinterpret_cast<T(*)[CW]>(al + k * CW));
  }

  T dov[NE], kv[NE];
  T delta;
  {
    T ov[NE];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      ld_own<T, CB>(a.dO + vrow + k * CW, *reinterpret_cast<T(*)[CW]>(dov + k * CW));
      ld_own<T, CB>(a.O + vrow + k * CW, *reinterpret_cast<T(*)[CW]>(ov + k * CW));
    }
    T s = T(0);
#pragma unroll
    for (int i = 0; i < NE; ++i) s += dov[i] * ov[i];
    delta = head_sum(s, lph);
  }
  const Rec<T> rec = ld_rec(a.stats, ri);  // m, ll2 of this row; aux = er | 1/||K||
  T erv = T(0), rk = T(1);
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.K + vrow + k * CW, *reinterpret_cast<T(*)[CW]>(kv + k * CW));
    if (a.l2) rk = rec.aux;
  } else {
    erv = rec.aux;
  }
  const T mrow = rec.m, ll2 = rec.ll2;

  T acc[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) acc[j] = T(0);

  constexpr int ep = pk ? 1 : EPW;
  const int js = pk ? 0 : sub;
  for (int base = eb; pk || base < ee; base += 32) {
    const int cnt = pk ? ee - eb : min(32, ee - base);
    const int cntw = pk ? static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(cnt))) : cnt;
    const int myu = nxt;
    if (!pk) {
      const int nb = base + 32;
      nxt = nb < ee ? (nb + lane < ee ? ld_idx(a.idx + nb + lane) : 0)
                    : (rsn.y + lane < rsn.z ? ld_idx(a.idx + rsn.y + lane) : 0);
    }
#if GF_FULL_CHUNK_A
    // whole 32-edge chunks: mask-free copy of the edge loop (as the forward)
    auto chunk = [&](auto full_tag, const int jb, const int je) {
      constexpr bool FULL = decltype(full_tag)::value;
  #pragma unroll 1
      for (int j0 = jb; j0 < je; j0 += ep * U) {
        bool ok[U];
        T vv[U][NE], qv[U][NE], el[U];
        int uus[U];
        // every slot's id first, then every gather: without the head_sum
        // branches (LPHC = 1) ptxas otherwise starts slot 0's math before
        // issuing slot 1's load, serialising the two L2 round trips
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;
          const int u = PKPRE ? __shfl_sync(kFull, myu, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myu, j & 31);
          uus[t] = ok[t] ? u : 0;
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int uu = uus[t];
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>(row_at(Vb, uu, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(vv[t] + k * CW), pol);
          if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(row_at(Qb, uu, qb) + k * CW, *reinterpret_cast<T(*)[CW]>(qv[t] + k * CW), pol);
          } else if constexpr (VAR == GF_ADDV) {
            el[t] = T(0);  // from the gathered V row below
          } else {
            el[t] = ld_node(row_at(Qb, uu, qb), pol);
          }
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          T dp = bdot<VAR != GF_ADDV>(dov, vv[t]);
          dp = head_sum(dp, lph);
          T s, rq = T(1), pre = T(0);
          if constexpr (VAR == GF_DOT) {
            T d = bdot<true>(qv[t], kv), qq = bdot<true>(qv[t], qv[t]);
            d = head_sum(d, lph);
            if (a.l2) {
              rq = inv_norm(head_sum(qq, lph));
              d *= rq * rk;
            }
            s = a.scale * d;
          } else {
            if constexpr (VAR == GF_ADDV) el[t] = head_sum(dot_n(vv[t], al), lph);
            pre = el[t] + erv;
            s = lrelu(pre, a.slope);
          }
          const T p = ok[t] ? ex2((s - mrow) * l2e<T>() - ll2) : T(0);
          const T ds = p * (dp - delta);
          if constexpr (VAR == GF_DOT) {
            const T w = a.scale * ds * rq;
  #pragma unroll
            for (int i = 0; i < NE; ++i) acc[i] += w * qv[t][i];
          } else {
            acc[0] += ds * lrelu_grad(pre, a.slope);
          }
        }
      }
    };
#if GF_FULL_STEPS
    // every step whose U slots all lie inside the chunk runs mask-free (rows
    // shorter than a chunk too); the remainder runs masked
    if (!pk && CPL == 1) {
      const int fe = cnt / (ep * U) * (ep * U);
      if (fe > 0) chunk(std::true_type{}, 0, fe);
      if (fe < cntw) chunk(std::false_type{}, fe, cntw);
    } else {
      chunk(std::false_type{}, 0, cntw);
    }
#else
    if (!pk && CPL == 1 && (32 % (EPW * U)) == 0 && cnt == 32)
      chunk(std::true_type{}, 0, cntw);
    else
      chunk(std::false_type{}, 0, cntw);
#endif
#else
    {
      constexpr bool FULL = false;
  #pragma unroll 1
      for (int j0 = 0; j0 < cntw; j0 += ep * U) {
        bool ok[U];
        T vv[U][NE], qv[U][NE], el[U];
        int uus[U];
        // every slot's id first, then every gather: without the head_sum
        // branches (LPHC = 1) ptxas otherwise starts slot 0's math before
        // issuing slot 1's load, serialising the two L2 round trips
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;
          const int u = PKPRE ? __shfl_sync(kFull, myu, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myu, j & 31);
          uus[t] = ok[t] ? u : 0;
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int uu = uus[t];
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>(row_at(Vb, uu, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(vv[t] + k * CW), pol);
          if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(row_at(Qb, uu, qb) + k * CW, *reinterpret_cast<T(*)[CW]>(qv[t] + k * CW), pol);
          } else if constexpr (VAR == GF_ADDV) {
            el[t] = T(0);  // from the gathered V row below
          } else {
            el[t] = ld_node(row_at(Qb, uu, qb), pol);
          }
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          T dp = bdot<VAR != GF_ADDV>(dov, vv[t]);
          dp = head_sum(dp, lph);
          T s, rq = T(1), pre = T(0);
          if constexpr (VAR == GF_DOT) {
            T d = bdot<true>(qv[t], kv), qq = bdot<true>(qv[t], qv[t]);
            d = head_sum(d, lph);
            if (a.l2) {
              rq = inv_norm(head_sum(qq, lph));
              d *= rq * rk;
            }
            s = a.scale * d;
          } else {
            if constexpr (VAR == GF_ADDV) el[t] = head_sum(dot_n(vv[t], al), lph);
            pre = el[t] + erv;
            s = lrelu(pre, a.slope);
          }
          const T p = ok[t] ? ex2((s - mrow) * l2e<T>() - ll2) : T(0);
          const T ds = p * (dp - delta);
          if constexpr (VAR == GF_DOT) {
            const T w = a.scale * ds * rq;
  #pragma unroll
            for (int i = 0; i < NE; ++i) acc[i] += w * qv[t][i];
          } else {
            acc[0] += ds * lrelu_grad(pre, a.slope);
          }
        }
      }
    }
#endif
    if (pk) break;
  }
  if (!pk && eb >= ee) nxt = rsn.y + lane < rsn.z ? ld_idx(a.idx + rsn.y + lane) : 0;

  if (!pk) warp_sum<T, LPE, NA>(acc);
  if (cta && !cta_sum<T, LPE, NA>(acc, warp, c, sub)) return;
  if (cta && ct.z > 1) {  // split row: the last CTA sums the slices in slice order
    if (!split_publish<NA>(a.part, a.part_cnt, ct, c, LPE, acc, sub == 0)) return;
    T x[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = T(0);
    for (int k = 0; k < ct.z; ++k) {
      split_load<NA>(a.part, ct, k, c, LPE, x);
#pragma unroll
      for (int j = 0; j < NA; ++j) acc[j] += x[j];
    }
  }
  const bool writer = pk ? live : sub == 0;

  if constexpr (VAR == GF_DOT) {
    if (a.l2) l2_backward_row<T, NE>(acc, kv, lph);
    if (writer) {
#pragma unroll
      for (int k = 0; k < CPL; ++k)
        st_chunk<T, CB>(a.dK + vrow + k * CW, *reinterpret_cast<T(*)[CW]>(acc + k * CW));
    }
  }
  if (writer && c % lph == 0) {
    a.stats[4 * ri + 3] = delta;
    if constexpr (VAR != GF_DOT) a.dK[ri] = acc[0];
  }
  rs = rsn;
  rsn = rsnn;
  }  // rows
}

// Bucket dispatch shared by both passes: CTA rows, warp rows, packed rows.
#define GF_BWD_DISPATCH(ROWFN)                                                                  \
  constexpr int EPW = 32 / LPE;                                                                 \
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;                                   \
  const int cb = a.cta_tab ? a.cta_blocks : a.n_cta;                                            \
  const int4 one = make_int4(0, 0, 1, -1);                                                      \
  if (blockIdx.x < static_cast<unsigned>(cb)) {                                                 \
    const int4 ct = a.cta_tab ? __ldg(a.cta_tab + blockIdx.x) : make_int4(blockIdx.x, 0, 1, -1); \
    ROWFN<T, CB, LPE, CPL, VAR, false>(a, lane, warp, true, ct.x, true, 1, ct);                 \
  } else if (blockIdx.x < static_cast<unsigned>(cb + a.wblocks)) {                              \
    const int slot = a.n_cta + ((blockIdx.x - cb) * kWarpsPerBlock + warp) * a.rpw;             \
    if (slot >= a.pk0) return;                                                                  \
    if (GF_BWD_LPH1 && CPL == 1 && (VAR == GF_ADDV || (GF_BWD_LPH1_TABLE && VAR == GF_ADD)) && a.LPH == 1) \
      ROWFN<T, CB, LPE, CPL, VAR, false, 1>(a, lane, warp, false, slot, true,                    \
                                            min(a.rpw, a.pk0 - slot), one);                     \
    else                                                                                        \
      ROWFN<T, CB, LPE, CPL, VAR, false>(a, lane, warp, false, slot, true,                       \
                                         min(a.rpw, a.pk0 - slot), one);                        \
  } else if constexpr (EPW > 1) {                                                               \
    const int slot = a.pk0 + ((blockIdx.x - cb - a.wblocks) * kWarpsPerBlock + warp) * EPW +    \
                     lane / LPE;                                                                \
    const bool live = slot < a.n;                                                               \
    if (!__any_sync(kFull, live)) return;                                                       \
    ROWFN<T, CB, LPE, CPL, VAR, true>(a, lane, warp, false, slot, live, 1, one);                \
  }

template <typename T, int CB, int LPE, int CPL, int VAR>
__global__ void __launch_bounds__(256, CPL == 1 ? (VAR == GF_ADDV ? GF_MINB_ROWS_V : GF_MINB_ROWS) : GF_MINB2) bwd_rows_fast(const BwdArgs<T> a) {
  pdl_launch();
  if (a.pf_len[0] > 0) l2_prefetch_tables(a.pf_ptr, a.pf_len);
  pdl_wait();
  GF_BWD_DISPATCH(bwd_row)
}

// ------------------------------------------------------------ pass B ------
template <typename T, int CB, int LPE, int CPL, int VAR, bool PK, int LPHC = 0>
__device__ __forceinline__ void bwd_col(const BwdArgs<T>& a, const int lane, const int warp,
                                        const bool cta, const int slot, const bool live,
                                        int /*nrows: pass B runs one column per warp, see below*/,
                                        const int4 ct) {
  const int lph = LPHC ? LPHC : a.LPH;
  constexpr int CW = Chunk<T, CB>::W;
  constexpr int NE = CPL * CW;
  constexpr int EPW = 32 / LPE;
  constexpr int U = CPL == 1 ? (VAR == GF_DOT ? GF_U_DOT1_COLS : GF_U_COLS) : (PK ? GF_U2_PK : GF_U2);
  constexpr int NT = NE + (VAR == GF_DOT ? NE : 1);  // dV chunk + (dQ chunk | del)
  constexpr bool pk = PK;  // packed column: this LPE-lane group owns the column
  const int c = lane % LPE, sub = lane / LPE;
  // No row pipelining / 16 B schedule entries here: at pass B's 64-register
  // budget (4 CTAs/SM) either spills; the launcher keeps rpw = 1.
  constexpr bool PKPRE = PK && LPE >= kSmallDegree;  // packed columns: sched entry + ids up front
  int u, sb, se;
  if constexpr (PK) {
    const int4 e = live ? ld_sched(a.sched + slot) : make_int4(0, 0, 0, 0);
    u = e.x, sb = e.y, se = e.z;
  } else {
    u = live ? __ldg(a.order + slot) : 0;
    sb = live ? __ldg(a.ptr + u) : 0, se = live ? __ldg(a.ptr + u + 1) : 0;
  }
  if (cta) {
    if (ct.z > 1) split_range(sb, se, ct.z, ct.y, sb, se);  // this CTA's slice of a split column
    split_range(sb, se, kWarpsPerBlock, warp, sb, se);
  }

  const int h = c / lph;
  const int off = h * a.D + (c % lph) * NE;
  const size_t urow = static_cast<size_t>(u) * a.F + off;
  const T* __restrict__ dOb = a.dO + off;
  const uint32_t fb = a.F * sizeof(T);
  const uint64_t pol = GF_POL_PARAM_BWD ? a.pol : pol_keep();
  const T* __restrict__ Kb = a.K + off;
  const T* __restrict__ Rb = a.stats + 4 * h;

  // Source-side operands owned by this column.
  T vu[NE], qu[NE];
  T elu = T(0), rq = T(1);
#pragma unroll
  for (int k = 0; k < CPL; ++k)
    ld_own<T, CB>(a.V + urow + k * CW, *reinterpret_cast<T(*)[CW]>(vu + k * CW));
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.Q + urow + k * CW, *reinterpret_cast<T(*)[CW]>(qu + k * CW));
    if (a.l2) {
      T s = T(0);
#pragma unroll
      for (int i = 0; i < NE; ++i) s += qu[i] * qu[i];
      rq = inv_norm(head_sum(s, lph));
    }
  } else if constexpr (VAR == GF_ADDV) {  // el = <V[u], a_l> from the owned V row
    T al[NE];
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.Q + off + k * CW, *reinterpret_cast<T(*)[CW]>(al + k * CW));
    elu = head_sum(dot_n(vu, al), lph);
  } else {
    elu = __ldg(a.Q + static_cast<size_t>(u) * a.H + h);
  }

  T all[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) all[j] = T(0);

  constexpr int ep = pk ? 1 : EPW;
  const int js = pk ? 0 : sub;
  int nxt = !pk && sb + lane < se ? ld_idx(a.idx + sb + lane) : 0;
  if constexpr (PKPRE) nxt = c < se - sb ? ld_idx(a.idx + sb + c) : 0;
  for (int base = sb; pk || base < se; base += 32) {
    const int cnt = pk ? se - sb : min(32, se - base);
    const int cntw = pk ? static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(cnt))) : cnt;
    const int myv = nxt;
    if (!pk) nxt = base + 32 + lane < se ? ld_idx(a.idx + base + 32 + lane) : 0;
#if GF_FULL_CHUNK_B
    // whole 32-edge chunks: mask-free copy of the edge loop (as the forward)
    auto chunk = [&](auto full_tag, const int jb, const int je) {
      constexpr bool FULL = decltype(full_tag)::value;
  #pragma unroll 1
      for (int j0 = jb; j0 < je; j0 += ep * U) {
        bool ok[U];
        T dov[U][NE], kv[U][NE];
        Rec<T> rec[U];
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;
          const int v = PKPRE ? __shfl_sync(kFull, myv, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myv, j & 31);
          const int vv = ok[t] ? v : 0;
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>(row_at(dOb, vv, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(dov[t] + k * CW), pol);
          if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(row_at(Kb, vv, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(kv[t] + k * CW), pol);
          }
          rec[t] = ld_rec(Rb, static_cast<size_t>(vv) * a.H);
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          T dp = bdot<true>(dov[t], vu);
          dp = head_sum(dp, lph);
          T s, rk = T(1), pre = T(0);
          if constexpr (VAR == GF_DOT) {
            T d = bdot<true>(qu, kv[t]);
            d = head_sum(d, lph);
            if (a.l2) {
              rk = rec[t].aux;
              d *= rq * rk;
            }
            s = a.scale * d;
          } else {
            pre = elu + rec[t].aux;
            s = lrelu(pre, a.slope);
          }
          const T p = ok[t] ? prob(s, rec[t]) : T(0);
          const T ds = p * (dp - rec[t].delta);
  #pragma unroll
          for (int i = 0; i < NE; ++i) all[i] += p * dov[t][i];
          if constexpr (VAR == GF_DOT) {
            const T w = a.scale * ds * rk;
  #pragma unroll
            for (int i = 0; i < NE; ++i) all[NE + i] += w * kv[t][i];
          } else {
            all[NE] += ds * lrelu_grad(pre, a.slope);
          }
        }
      }
    };
#if GF_FULL_STEPS
    // every step whose U slots all lie inside the chunk runs mask-free (rows
    // shorter than a chunk too); the remainder runs masked
    if (!pk && CPL == 1) {
      const int fe = cnt / (ep * U) * (ep * U);
      if (fe > 0) chunk(std::true_type{}, 0, fe);
      if (fe < cntw) chunk(std::false_type{}, fe, cntw);
    } else {
      chunk(std::false_type{}, 0, cntw);
    }
#else
    if (!pk && CPL == 1 && (32 % (EPW * U)) == 0 && cnt == 32)
      chunk(std::true_type{}, 0, cntw);
    else
      chunk(std::false_type{}, 0, cntw);
#endif
#else
    {
      constexpr bool FULL = false;
  #pragma unroll 1
      for (int j0 = 0; j0 < cntw; j0 += ep * U) {
        bool ok[U];
        T dov[U][NE], kv[U][NE];
        Rec<T> rec[U];
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;
          const int v = PKPRE ? __shfl_sync(kFull, myv, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myv, j & 31);
          const int vv = ok[t] ? v : 0;
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>(row_at(dOb, vv, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(dov[t] + k * CW), pol);
          if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(row_at(Kb, vv, fb) + k * CW, *reinterpret_cast<T(*)[CW]>(kv[t] + k * CW), pol);
          }
          rec[t] = ld_rec(Rb, static_cast<size_t>(vv) * a.H);
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          T dp = bdot<true>(dov[t], vu);
          dp = head_sum(dp, lph);
          T s, rk = T(1), pre = T(0);
          if constexpr (VAR == GF_DOT) {
            T d = bdot<true>(qu, kv[t]);
            d = head_sum(d, lph);
            if (a.l2) {
              rk = rec[t].aux;
              d *= rq * rk;
            }
            s = a.scale * d;
          } else {
            pre = elu + rec[t].aux;
            s = lrelu(pre, a.slope);
          }
          const T p = ok[t] ? prob(s, rec[t]) : T(0);
          const T ds = p * (dp - rec[t].delta);
  #pragma unroll
          for (int i = 0; i < NE; ++i) all[i] += p * dov[t][i];
          if constexpr (VAR == GF_DOT) {
            const T w = a.scale * ds * rk;
  #pragma unroll
            for (int i = 0; i < NE; ++i) all[NE + i] += w * kv[t][i];
          } else {
            all[NE] += ds * lrelu_grad(pre, a.slope);
          }
        }
      }
    }
#endif
    if (pk) break;
  }

  if (!pk) warp_sum<T, LPE, NT>(all);
  if (cta && !cta_sum<T, LPE, NT>(all, warp, c, sub)) return;
  if (cta && ct.z > 1) {  // split column: the last CTA sums the slices in slice order
    if (!split_publish<NT>(a.part, a.part_cnt, ct, c, LPE, all, sub == 0)) return;
    T x[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) all[j] = T(0);
    for (int k = 0; k < ct.z; ++k) {
      split_load<NT>(a.part, ct, k, c, LPE, x);
#pragma unroll
      for (int j = 0; j < NT; ++j) all[j] += x[j];
    }
  }

  T g[NE];
  if constexpr (VAR == GF_DOT) {
#pragma unroll
    for (int i = 0; i < NE; ++i) g[i] = all[NE + i];
    if (a.l2) l2_backward_row<T, NE>(g, qu, lph);
  }
  if (pk ? live : sub == 0) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      st_chunk<T, CB>(a.dV + urow + k * CW, *reinterpret_cast<T(*)[CW]>(all + k * CW));
      if constexpr (VAR == GF_DOT)
        st_chunk<T, CB>(a.dQ + urow + k * CW, *reinterpret_cast<T(*)[CW]>(g + k * CW));
    }
    if constexpr (VAR != GF_DOT) {
      if (c % lph == 0) a.dQ[static_cast<size_t>(u) * a.H + h] = all[NE];
    }
  }
}

template <typename T, int CB, int LPE, int CPL, int VAR>
__global__ void __launch_bounds__(256, CPL == 1 ? (VAR == GF_DOT ? GF_MINB_DOT1_COLS : GF_MINB_COLS) : GF_MINB2) bwd_cols_fast(const BwdArgs<T> a) {
  // one call site for CTA and warp columns (runtime `cta`): two inlined copies
  // push pass B past its 64-register budget
  pdl_launch();
  if (a.pf_len[0] > 0) l2_prefetch_tables(a.pf_ptr, a.pf_len);
  pdl_wait();
  constexpr int EPW = 32 / LPE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cb = a.cta_tab ? a.cta_blocks : a.n_cta;
  const bool cta = blockIdx.x < static_cast<unsigned>(cb);
  if (cta || blockIdx.x < static_cast<unsigned>(cb + a.wblocks)) {
    const int4 ct = !cta ? make_int4(0, 0, 1, -1)
                         : (a.cta_tab ? __ldg(a.cta_tab + blockIdx.x) : make_int4(blockIdx.x, 0, 1, -1));
    const int slot = cta ? ct.x : a.n_cta + (blockIdx.x - cb) * kWarpsPerBlock + warp;
    if (!cta && slot >= a.pk0) return;
    if (GF_BWDC_LPH1 && CPL == 1 && (VAR == GF_ADDV || (GF_BWD_LPH1_TABLE && VAR == GF_ADD)) && !cta &&
        a.LPH == 1)
      bwd_col<T, CB, LPE, CPL, VAR, false, 1>(a, lane, warp, false, slot, true, 1, ct);
    else
      bwd_col<T, CB, LPE, CPL, VAR, false>(a, lane, warp, cta, slot, true, 1, ct);
  } else if constexpr (EPW > 1) {
    const int slot = a.pk0 + ((blockIdx.x - cb - a.wblocks) * kWarpsPerBlock + warp) * EPW +
                     lane / LPE;
    const bool live = slot < a.n;
    if (!__any_sync(kFull, live)) return;
    bwd_col<T, CB, LPE, CPL, VAR, true>(a, lane, warp, false, slot, live, 1, make_int4(0, 0, 1, -1));
  }
}

// ----------------------------------------------------------- generic path --
// Serial-per-head versions for shapes that do not tile into 16/32-byte chunks.
template <typename T, int VAR>
__global__ void __launch_bounds__(128) bwd_rows_generic(const BwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * kGenericWarps + warp;
  if (slot >= a.n) return;
  T* ws = reinterpret_cast<T*>(smraw) + static_cast<size_t>(warp) * (3 * a.F + 32);
  T* dos = ws;           // dO[v]
  T* kvs = ws + a.F;     // K[v]
  T* gk = ws + 2 * a.F;  // dKhat[v]
  T* wh = ws + 3 * a.F;  // per-head edge weight
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
  T dlt = T(0), gr = T(0);
  Rec<T> rec{};
  if (lane < a.H) {
    for (int j = 0; j < a.D; ++j) dlt += dos[lane * a.D + j] * __ldg(a.O + vrow + lane * a.D + j);
    a.stats[4 * (static_cast<size_t>(v) * a.H + lane) + 3] = dlt;
    rec = ld_rec(a.stats, static_cast<size_t>(v) * a.H + lane);
  }
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    if (lane < a.H) {
      T rq = T(1), pre = T(0);
      const T s = generic_score<T, VAR>(a, u, v, lane, kvs, erh, rkh, &rq, &pre);
      const T p = prob(s, rec);
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
      const Rec<T> rec = ld_rec(a.stats, static_cast<size_t>(v) * a.H + lane);
      T s, pre = T(0), rk = T(1);
      if constexpr (VAR == GF_DOT) {
        T d = T(0);
        for (int j = 0; j < a.D; ++j) d += qus[lane * a.D + j] * __ldg(a.K + vrow + lane * a.D + j);
        if (a.l2) {
          rk = rec.aux;
          s = a.scale * d * (rqh * rk);
        } else {
          s = a.scale * d;
        }
      } else {
        pre = elh + rec.aux;
        s = lrelu(pre, a.slope);
      }
      const T p = prob(s, rec);
      T dp = T(0);
      for (int j = 0; j < a.D; ++j) dp += __ldg(a.dO + vrow + lane * a.D + j) * vus[lane * a.D + j];
      const T ds = p * (dp - rec.delta);
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

template <typename T, int CB, int LPE, int CPL>
int launch_fast_bwd(const BwdArgs<T>& ra, const BwdArgs<T>& ca, int variant, int rblocks,
                    int cblocks, cudaStream_t s) {
  if (variant == GF_DOT) {
    if (rblocks) GF_CHECK_CUDA(launch_k(bwd_rows_fast<T, CB, LPE, CPL, GF_DOT>, rblocks, 256, s, ra));
    GF_CHECK_LAUNCH("bwd_rows_fast");
    if (cblocks) GF_CHECK_CUDA(launch_k(bwd_cols_fast<T, CB, LPE, CPL, GF_DOT>, cblocks, 256, s, ca));
    GF_CHECK_LAUNCH("bwd_cols_fast");
  } else if (variant == GF_ADDV) {
    if (rblocks) GF_CHECK_CUDA(launch_k(bwd_rows_fast<T, CB, LPE, CPL, GF_ADDV>, rblocks, 256, s, ra));
    GF_CHECK_LAUNCH("bwd_rows_fast");
    if (cblocks) GF_CHECK_CUDA(launch_k(bwd_cols_fast<T, CB, LPE, CPL, GF_ADDV>, cblocks, 256, s, ca));
    GF_CHECK_LAUNCH("bwd_cols_fast");
  } else {
    if (rblocks) GF_CHECK_CUDA(launch_k(bwd_rows_fast<T, CB, LPE, CPL, GF_ADD>, rblocks, 256, s, ra));
    GF_CHECK_LAUNCH("bwd_rows_fast");
    if (cblocks) GF_CHECK_CUDA(launch_k(bwd_cols_fast<T, CB, LPE, CPL, GF_ADD>, cblocks, 256, s, ca));
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

bool aligned(const void* p, int b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; }

}  // namespace

template <typename T>
int launch_bwd(const DevGraph& g, BwdArgs<T> a, int variant, int passes, cudaStream_t s) {
  if (g.n == 0) return GF_OK;
  BwdArgs<T> ra = a, ca = a;
  ra.ptr = g.row_ptr, ra.idx = g.col, ra.order = g.row_order, ra.n_cta = g.n_cta_rows;
  ca.ptr = g.csc_ptr, ca.idx = g.csc_row, ca.order = g.col_order, ca.n_cta = g.n_cta_cols;
  ra.cta_tab = g.row_cta, ra.cta_blocks = g.row_cta_blocks, ra.parts = g.row_parts;
  ca.cta_tab = g.col_cta, ca.cta_blocks = g.col_cta_blocks, ca.parts = g.col_parts;
  ra.sched = g.row_sched, ca.sched = g.col_sched;
  ra.n = g.active_rows();
  ca.n = g.active_cols();
  const bool do_a = passes & 1, do_b = passes & 2;
  const bool dot = variant == GF_DOT;
  // Each pass picks the fast path independently (both paths use the same
  // record layout), so a misaligned operand of one pass never affects the other.
  const FastShape fs = fast_shape(a.H, a.D, sizeof(T), g.e);
  const int cb = fs.cb;
  const bool base = fs.ok && static_cast<int64_t>(g.n) * a.F < (int64_t(1) << 31) &&
                    aligned(a.stats, 32);
  const bool addv = variant == GF_ADDV;
  const bool fast_a = base && aligned(a.V, cb) && aligned(a.O, 16) && aligned(a.dO, 16) &&
                      (!dot || (aligned(a.Q, cb) && aligned(a.K, 16) && aligned(a.dK, 16))) &&
                      (!addv || aligned(a.Q, cb));
  const bool fast_b = base && aligned(a.V, 16) && aligned(a.dO, cb) && aligned(a.dV, 16) &&
                      (!dot || (aligned(a.Q, 16) && aligned(a.K, cb) && aligned(a.dQ, 16))) &&
                      (!addv || aligned(a.Q, cb));
  if (addv && ((do_a && !fast_a) || (do_b && !fast_b))) {
    set_error("gf_attn_bwd: logits-from-V needs the fast path (callers fall back to el/er tables)");
    return GF_ERR_INVALID;
  }
  ra.LPH = ca.LPH = fs.ok ? fs.lph : 1;
  // bucket geometry (see fwd): warp bucket [n_cta, pk0), packed [pk0, n)
  const int epw = fs.ok ? 32 / fs.lpe : 1;
  // warp rows per warp: 8 for short rows (average degree <= 64), else 1 (as fwd)
  ca.rpw = 1;  // pass B: no row pipelining (register budget, see bwd_col)
  auto buckets = [&](BwdArgs<T>& x, int n_small, int n_empty) {
    x.pk0 = epw > 1 ? std::max(x.n_cta, g.n - n_empty - n_small) : x.n;
    x.pk0 = std::min(x.pk0, x.n);
    if (&x == &ra) x.rpw = rows_per_warp(g.e, g.n, x.pk0 - x.n_cta);
    x.wblocks = (x.pk0 - x.n_cta + kWarpsPerBlock * x.rpw - 1) / (kWarpsPerBlock * x.rpw);
    const int per_block = kWarpsPerBlock * epw;
    const int cta_blocks = x.cta_tab ? x.cta_blocks : x.n_cta;
    return cta_blocks + x.wblocks + (x.n - x.pk0 + per_block - 1) / per_block;
  };
  const int rb = (do_a && fast_a) ? buckets(ra, g.n_small_rows, g.n_empty_rows) : 0;
  const int cbk = (do_b && fast_b) ? buckets(ca, g.n_small_cols, g.n_empty_cols) : 0;
  // small graphs: prefetch each pass's gathered tables into L2 at entry
  // (pass A: V, Q|el, dO; pass B: dO, K (dot), the records)
  if (l2_prefetch_enabled() && g.e < kPrefetchMaxEdges) {
    const int64_t fb = static_cast<int64_t>(g.n) * a.F * static_cast<int64_t>(sizeof(T));
    const int64_t qb = dot ? fb : is_addv(variant) ? 0 : static_cast<int64_t>(g.n) * a.H * sizeof(T);
    const int64_t rb = static_cast<int64_t>(g.n) * a.H * 4 * static_cast<int64_t>(sizeof(T));
    if (2 * fb + qb <= kPrefetchMaxBytes) {
      ra.pf_ptr[0] = a.V, ra.pf_len[0] = fb;
      ra.pf_ptr[1] = a.Q, ra.pf_len[1] = qb;
      ra.pf_ptr[2] = a.dO, ra.pf_len[2] = fb;
    }
    if (fb + (dot ? fb : 0) + rb <= kPrefetchMaxBytes) {
      ca.pf_ptr[0] = a.dO, ca.pf_len[0] = fb;
      ca.pf_ptr[1] = a.K, ca.pf_len[1] = dot ? fb : 0;
      ca.pf_ptr[2] = a.stats, ca.pf_len[2] = rb;
    }
  }
  // split super rows / columns: slice partials + arrival counters
  const size_t ne = fs.ok ? static_cast<size_t>(fs.cpl) * (fs.cb / sizeof(T)) : 0;
  auto parts = [&](BwdArgs<T>& x, size_t nv) -> int {
    if (!x.cta_tab || x.parts == 0) return GF_OK;
    GF_CHECK_CUDA(scratch_alloc(&x.part, sizeof(T) * x.parts * fs.lpe * nv, s));
    GF_CHECK_CUDA(scratch_alloc(&x.part_cnt, sizeof(unsigned) * x.parts, s));
    GF_CHECK_CUDA(cudaMemsetAsync(x.part_cnt, 0, sizeof(unsigned) * x.parts, s));
    return GF_OK;
  };
  struct PartFree {
    BwdArgs<T>& r;
    BwdArgs<T>& c;
    cudaStream_t s;
    ~PartFree() {
      for (BwdArgs<T>* x : {&r, &c}) {
        if (x->part) cudaFreeAsync(x->part, s);
        if (x->part_cnt) cudaFreeAsync(x->part_cnt, s);
      }
    }
  } part_free{ra, ca, s};
  if (rb) {
    if (int rc = parts(ra, dot ? ne : 1)) return rc;
  }
  if (cbk) {
    if (int rc = parts(ca, ne + (dot ? ne : 1))) return rc;
  }
  if (rb || cbk) {
    int rc = GF_OK;
    switch (fs.cb * 1000 + fs.lpe * 10 + fs.cpl) {
      case 32011: rc = launch_fast_bwd<T, 32, 1, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32021: rc = launch_fast_bwd<T, 32, 2, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32041: rc = launch_fast_bwd<T, 32, 4, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32081: rc = launch_fast_bwd<T, 32, 8, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32161: rc = launch_fast_bwd<T, 32, 16, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32321: rc = launch_fast_bwd<T, 32, 32, 1>(ra, ca, variant, rb, cbk, s); break;
      case 32012: rc = launch_fast_bwd<T, 32, 1, 2>(ra, ca, variant, rb, cbk, s); break;
      case 32022: rc = launch_fast_bwd<T, 32, 2, 2>(ra, ca, variant, rb, cbk, s); break;
      case 32042: rc = launch_fast_bwd<T, 32, 4, 2>(ra, ca, variant, rb, cbk, s); break;
      case 32082: rc = launch_fast_bwd<T, 32, 8, 2>(ra, ca, variant, rb, cbk, s); break;
      case 32162: rc = launch_fast_bwd<T, 32, 16, 2>(ra, ca, variant, rb, cbk, s); break;
      case 32322: rc = launch_fast_bwd<T, 32, 32, 2>(ra, ca, variant, rb, cbk, s); break;
      case 16011: rc = launch_fast_bwd<T, 16, 1, 1>(ra, ca, variant, rb, cbk, s); break;
      case 16021: rc = launch_fast_bwd<T, 16, 2, 1>(ra, ca, variant, rb, cbk, s); break;
      case 16041: rc = launch_fast_bwd<T, 16, 4, 1>(ra, ca, variant, rb, cbk, s); break;
      case 16081: rc = launch_fast_bwd<T, 16, 8, 1>(ra, ca, variant, rb, cbk, s); break;
      case 16161: rc = launch_fast_bwd<T, 16, 16, 1>(ra, ca, variant, rb, cbk, s); break;
      case 16321: rc = launch_fast_bwd<T, 16, 32, 1>(ra, ca, variant, rb, cbk, s); break;
      default: set_error("gf_attn_bwd: internal fast-shape dispatch"); return GF_ERR_CUDA;
    }
    if (rc) return rc;
  }
  const bool gen_a = do_a && !fast_a && ra.n > 0, gen_b = do_b && !fast_b && ca.n > 0;
  if (!gen_a && !gen_b) return GF_OK;
  if (a.H > 32) {
    set_error("gf_attn_bwd: heads > 32 need a head shape that tiles into 16/32-byte chunks");
    return GF_ERR_UNSUPPORTED;
  }
  const size_t sa = static_cast<size_t>(kGenericWarps) * (3 * a.F + 32) * sizeof(T);
  const size_t sbm = static_cast<size_t>(kGenericWarps) * (4 * a.F + 64) * sizeof(T);
  if (sbm > 200 * 1024) {
    set_error("gf_attn_bwd: feature width too large for the generic path");
    return GF_ERR_UNSUPPORTED;
  }
  const int rblk = (ra.n + kGenericWarps - 1) / kGenericWarps;
  const int cblk = (ca.n + kGenericWarps - 1) / kGenericWarps;
  int rc;
  if (dot) {
    if (gen_a) {
      if ((rc = set_smem(bwd_rows_generic<T, GF_DOT>, sa))) return rc;
      bwd_rows_generic<T, GF_DOT><<<rblk, 32 * kGenericWarps, sa, s>>>(ra);
      GF_CHECK_LAUNCH("bwd_rows_generic");
    }
    if (gen_b) {
      if ((rc = set_smem(bwd_cols_generic<T, GF_DOT>, sbm))) return rc;
      bwd_cols_generic<T, GF_DOT><<<cblk, 32 * kGenericWarps, sbm, s>>>(ca);
      GF_CHECK_LAUNCH("bwd_cols_generic");
    }
  } else {
    if (gen_a) {
      if ((rc = set_smem(bwd_rows_generic<T, GF_ADD>, sa))) return rc;
      bwd_rows_generic<T, GF_ADD><<<rblk, 32 * kGenericWarps, sa, s>>>(ra);
      GF_CHECK_LAUNCH("bwd_rows_generic");
    }
    if (gen_b) {
      if ((rc = set_smem(bwd_cols_generic<T, GF_ADD>, sbm))) return rc;
      bwd_cols_generic<T, GF_ADD><<<cblk, 32 * kGenericWarps, sbm, s>>>(ca);
      GF_CHECK_LAUNCH("bwd_cols_generic");
    }
  }
  return GF_OK;
}

}  // namespace gfb

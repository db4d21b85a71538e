#pragma once
// (Included by gf_attn_fwd_f32.cu / gf_attn_fwd_f64.cu: one translation unit
// per element type so the two halves of the kernel instantiations compile in
// parallel.)
//
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
//     schedule.cpp:42-60), each warp runs an online (max, sum) softmax over
//     its slice in registers, and the 8 partial states are merged in shared
//     memory in a fixed order (deterministic);
//   * every other row is warp-per-row.
// Lane mapping: a lane owns (a 2-chunk slice of) ONE head and gathers it with
// 256-bit loads (LDG.E.256, one full 32 B sector per lane), so per-head score
// / softmax work is done once per edge, not once per 16 B chunk; 32/LPE edges
// per warp step, unrolled U deep.  Nothing of size E x H is written: outputs
// are O (N x F) and the per-(row, head) softmax records (gf_device.cuh Rec).
#include <cstdlib>
#include <type_traits>

#include "gf_device.cuh"
#include "gf_internal.cuh"

#ifndef GF_FULL_CHUNK
#define GF_FULL_CHUNK 1
#endif

#ifndef GF_WIDE_ADDR_FWD
#define GF_WIDE_ADDR_FWD 1  // 1: V rows of the layer form / MODE 2-3 as one IMAD.WIDE.U32 (C4 fwd -1.5 %)
#endif

#ifndef GF_RESCALE_TH
#define GF_RESCALE_TH 8  // natural-log units; 0 = rescale whenever a running max moves
#endif

#ifndef GF_FWD_LPH1
#define GF_FWD_LPH1 1  // GAT layer-form warp rows with one lane per head: LPH = 1 at compile time
#endif

#ifndef GF_FWD_LPH1_TABLE
#define GF_FWD_LPH1_TABLE 0  // the same for the el / er table form (measured 6 % slower before the id hoist)
#endif

#ifndef GF_FWD_DOT2
#define GF_FWD_DOT2 1
#endif

#ifndef GF_FMAX
#define GF_FMAX 1  // running max as FMNMX (same NaN handling as the compare-select)
#endif

#ifndef GF_FULL_STEPS
#define GF_FULL_STEPS 0
#endif

namespace gfb {

namespace {

template <typename T, int N>
__device__ __forceinline__ void merge_state(T& m, T& l, T (&acc)[N], T m2, T l2,
                                            const T (&acc2)[N]) {
  const T mn = m > m2 ? m : m2;
  if (!(mn > ninf<T>())) return;  // both empty
  const T ca = expd(m - mn), cb = expd(m2 - mn);
  l = l * ca + l2 * cb;
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = acc[i] * ca + acc2[i] * cb;
  m = mn;
}

// MODE 0: SMMF (scores computed here); 1: PMF's fused softmax + SpMM over the
// scores an edge-parallel SDDMM wrote to a.ES; 2: the unfused SpMM (a.ES holds
// normalised probabilities: O = sum p V, no softmax, no records).
// Rows slot .. slot+nrows-1 (a CTA slice, nrows warp rows, or — PK — one
// packed row per LPE-lane group).  Warp rows are software-pipelined: the
// schedule entry two rows ahead and the next row's first 32 ids are loaded
// while the current row's gathers are in flight, so consecutive rows do not
// each pay the id round trip before their first gather.
template <typename T, int CB, int LPE, int CPL, int VAR, int MODE, bool PK, int LPHC = 0>
__device__ __forceinline__ void fwd_row(const FwdArgs<T>& a, const int lane, const int warp,
                                        const bool cta, const int slot, const bool live,
                                        const int nrows, const int4 ct) {
  // lanes per head: compile-time for the hot one-lane-per-head rows (LPHC = 1:
  // no head_sum loop guard and no reload of the runtime value per iteration)
  const int lph = LPHC ? LPHC : a.LPH;
  constexpr int CW = Chunk<T, CB>::W;
  constexpr int NE = CPL * CW;  // elements per lane
  constexpr int EPW = 32 / LPE;
  constexpr int U = CPL == 1 ? (VAR == GF_ADDV_HBM ? GF_U_FWD_H : VAR == GF_ADDV ? GF_U_FWD_V
                                : VAR == GF_DOT && MODE == 0 ? GF_U_DOT1 : GF_U_FWD)
                             : (PK ? GF_U2_PK : GF_U2);
  const int c = lane % LPE, sub = lane / LPE;
  constexpr bool pk = PK;
  const int4 zero4 = make_int4(0, 0, 0, 0);
  // Packed rows (degree <= kSmallDegree): the 16 B schedule entry (one load
  // instead of order -> pointers), and each lane group loads its row's ids
  // once up front (one id per lane) instead of one dependent load per edge.
  constexpr bool PKPRE = PK && LPE >= kSmallDegree;
  int4 rs;
  if constexpr (GF_SCHED16_FWD || PK) {
    rs = live ? ld_sched(a.sched + slot) : zero4;
  } else {
    const int v0 = live ? __ldg(a.order + slot) : 0;
    rs = live ? make_int4(v0, __ldg(a.ptr + v0), __ldg(a.ptr + v0 + 1), 0) : zero4;
  }
  int4 rsn = GF_ROWPIPE && nrows > 1 ? ld_sched(a.sched + slot + 1) : zero4;
  int nxt = 0;

  const int h = c / lph;
  const int off = h * a.D + (c % lph) * NE;  // first element owned by this lane
  const T* __restrict__ Vb = a.V + off;
  const T* __restrict__ Qb = a.Q + (VAR == GF_DOT ? off : h);
  const int qs = VAR == GF_DOT ? a.F : a.H;  // row stride of Q|el
  T al[NE];  // GF_ADDV: this lane's slice of a_l (el = <V[u], a_l> per head)
  if constexpr (is_addv(VAR)) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.Q + off + k * CW, *reinterpret_cast<T(*)[CW]>(al + k * CW));
  }
  const T* __restrict__ Sb = a.ES + h;        // MODE 1/2: ES[e * H + h]
  const uint64_t pol = GF_POL_PARAM_FWD ? a.pol : pol_keep();
  // V rows addressed as base + u * stride (one IMAD.WIDE.U32) where V is the
  // only gathered table (GAT layer form, MODE 2/3) or everywhere (= 2)
  constexpr bool WIDE = GF_WIDE_ADDR_FWD == 2 || (GF_WIDE_ADDR_FWD == 1 && (is_addv(VAR) || MODE >= 2));
  const uint32_t fb = static_cast<uint32_t>(a.F * sizeof(T));

  for (int r = 0; r < (GF_ROWPIPE ? nrows : 1); ++r) {
  const int4 rsnn = GF_ROWPIPE && r + 2 < nrows ? ld_sched(a.sched + slot + r + 2) : zero4;
  const int v = rs.x;
  int eb = rs.y, ee = rs.z;
  if (cta) {
    if (ct.z > 1) split_range(eb, ee, ct.z, ct.y, eb, ee);  // this CTA's slice of a split row
    split_range(eb, ee, kWarpsPerBlock, warp, eb, ee);
  }
  if (r == 0 && !pk) nxt = eb + lane < ee ? ld_idx(a.idx + eb + lane) : 0;
  if constexpr (PKPRE) nxt = c < ee - eb ? ld_idx(a.idx + eb + c) : 0;

  // Destination-side operands stay in registers for the whole row.
  T kv[NE];
  T erv = T(0), rk = T(1);
  if constexpr (MODE >= 2) {
    // probabilities given: no destination-side score operands
  } else if constexpr (VAR == GF_DOT) {
    if (MODE == 0 || a.l2) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      ld_own<T, CB>(a.K + static_cast<size_t>(v) * a.F + off + k * CW,
                    *reinterpret_cast<T(*)[CW]>(kv + k * CW));
    if (a.l2) {
      T s = T(0);
#pragma unroll
      for (int i = 0; i < NE; ++i) s += kv[i] * kv[i];
      rk = inv_norm(head_sum(s, lph));
    }
    }
  } else if constexpr (is_addv(VAR)) {  // er = <V[v], a_r> from the row's own V
    T vo[NE], ar[NE];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      ld_own<T, CB>(a.V + static_cast<size_t>(v) * a.F + off + k * CW,
                    *reinterpret_cast<T(*)[CW]>(vo + k * CW));
      ld_own<T, CB>(a.K + off + k * CW, *reinterpret_cast<T(*)[CW]>(ar + k * CW));
    }
    erv = head_sum(dot_n(vo, ar), lph);
  } else {
    erv = __ldg(a.K + static_cast<size_t>(v) * a.H + h);
  }

  T m = ninf<T>(), l = T(0), acc[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) acc[i] = T(0);

  // Warp / CTA rows: 32 ids per chunk, one per lane, shuffled to the edge
  // slots (next chunk prefetched); packed rows: each group walks its own
  // <= kSmallDegree edges one per step, loading ids directly.
  constexpr int ep = pk ? 1 : EPW;
  const int js = pk ? 0 : sub;
  for (int base = eb; pk || base < ee; base += 32) {
    const int cnt = pk ? ee - eb : min(32, ee - base);
    const int cntw = pk ? static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(cnt))) : cnt;
    const int myu = nxt;  // ids of this 32-edge chunk; prefetch the next one (or the next row's first)
    if (!pk) {
      const int nb = base + 32;
      nxt = nb < ee ? (nb + lane < ee ? ld_idx(a.idx + nb + lane) : 0)
                    : (rsn.y + lane < rsn.z ? ld_idx(a.idx + rsn.y + lane) : 0);
    }
#if GF_FULL_CHUNK
    // Whole 32-edge chunks (all but a row's last) run a mask-free copy of the
    // loop: no per-slot bounds compare / select on the ids and probabilities.
    auto chunk = [&](auto full_tag, const int jb, const int je) {
      constexpr bool FULL = decltype(full_tag)::value;
  #pragma unroll 1
      for (int j0 = jb; j0 < je; j0 += ep * U) {
        bool ok[U];
        T vv[U][NE], qv[U][NE], s[U];
        int uus[U];
        // every slot's id before any gather (as pass A: keeps ptxas from
        // starting slot 0's math ahead of the later slots' loads)
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;  // FULL: a whole 32-edge chunk, no masks
          const int u = PKPRE ? __shfl_sync(kFull, myu, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myu, j & 31);
          uus[t] = ok[t] ? u : 0;  // in-range dummy row for masked lanes
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          const int uu = uus[t];
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>((WIDE ? row_at(Vb, uu, fb) : Vb + uu * a.F) + k * CW, *reinterpret_cast<T(*)[CW]>(vv[t] + k * CW), pol);
          if constexpr (MODE == 3) {
            s[t] = ok[t] ? ld_edge(Sb + static_cast<size_t>(ld_idx(a.eperm + base + j)) * a.H) : T(0);
          } else if constexpr (MODE != 0) {
            s[t] = ok[t] ? ld_edge(Sb + static_cast<size_t>(base + j) * a.H) : T(0);
          } else if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(Qb + uu * qs + k * CW, *reinterpret_cast<T(*)[CW]>(qv[t] + k * CW), pol);
          } else if constexpr (is_addv(VAR)) {
            // el from the gathered V row (after the slot loop)
          } else {
            s[t] = ld_node(Qb + uu * qs, pol);
          }
        }
        if constexpr (MODE >= 2) {
  #pragma unroll
          for (int t = 0; t < U; ++t) {
            axpy_n(acc, s[t], vv[t]);
          }
          continue;
        }
        T smax = ninf<T>();
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          if constexpr (MODE == 1) {
            // score read from ES
          } else if constexpr (VAR == GF_DOT) {
            T d, qq;
            if constexpr (GF_FWD_DOT2) {  // paired FFMA2: half the dependent chain
              d = dot_n(qv[t], kv);
              qq = dot_n(qv[t], qv[t]);
            } else {
              d = T(0), qq = T(0);
  #pragma unroll
              for (int i = 0; i < NE; ++i) {
                d += qv[t][i] * kv[i];
                qq += qv[t][i] * qv[t][i];
              }
            }
            d = head_sum(d, lph);
            if (a.l2) d *= inv_norm(head_sum(qq, lph)) * rk;
            s[t] = a.scale * d;
          } else if constexpr (is_addv(VAR)) {
            s[t] = lrelu(head_sum(dot_n(vv[t], al), lph) + erv, a.slope);
          } else {
            s[t] = lrelu(s[t] + erv, a.slope);
          }
          s[t] = ok[t] ? s[t] : ninf<T>();
          smax = GF_FMAX ? fmax(s[t], smax) : (s[t] > smax ? s[t] : smax);
        }
        // Lazy rescale, warp-uniform: only when some lane's running max moves
        // past m + GF_RESCALE_TH.  Below that the stale m is kept: p = e^(s-m)
        // stays <= e^TH, and (m, l) remain a consistent pair (P = e^(s-m) / l
        // for any m), so records, merges and the backward are unchanged.
        if (__any_sync(kFull, smax > m + T(GF_RESCALE_TH))) {
          const T mn = smax > m ? smax : m;
          const T corr = m == mn ? T(1) : expd(m - mn);
          l *= corr;
          scale_n(acc, corr);
          m = mn;
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const T p = ok[t] ? expd(s[t] - m) : T(0);
          l += p;
          axpy_n(acc, p, vv[t]);
        }
      }
    };
    // (only when the loop's slots tile the chunk exactly — EPW * U divides 32 —
    // and for one-chunk lanes: the CPL = 2 shapes (GT 8x16) measured slower)
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
        T vv[U][NE], qv[U][NE], s[U];
        int uus[U];
        // every slot's id before any gather (as pass A: keeps ptxas from
        // starting slot 0's math ahead of the later slots' loads)
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          ok[t] = FULL || j < cnt;  // FULL: a whole 32-edge chunk, no masks
          const int u = PKPRE ? __shfl_sync(kFull, myu, (lane & ~(LPE - 1)) + (j & (LPE - 1)))
                        : pk ? (ok[t] ? ld_idx(a.idx + base + j) : 0) : __shfl_sync(kFull, myu, j & 31);
          uus[t] = ok[t] ? u : 0;  // in-range dummy row for masked lanes
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const int j = j0 + t * ep + js;
          const int uu = uus[t];
  #pragma unroll
          for (int k = 0; k < CPL; ++k)
            ld_gather<T, CB>((WIDE ? row_at(Vb, uu, fb) : Vb + uu * a.F) + k * CW, *reinterpret_cast<T(*)[CW]>(vv[t] + k * CW), pol);
          if constexpr (MODE == 3) {
            s[t] = ok[t] ? ld_edge(Sb + static_cast<size_t>(ld_idx(a.eperm + base + j)) * a.H) : T(0);
          } else if constexpr (MODE != 0) {
            s[t] = ok[t] ? ld_edge(Sb + static_cast<size_t>(base + j) * a.H) : T(0);
          } else if constexpr (VAR == GF_DOT) {
  #pragma unroll
            for (int k = 0; k < CPL; ++k)
              ld_gather<T, CB>(Qb + uu * qs + k * CW, *reinterpret_cast<T(*)[CW]>(qv[t] + k * CW), pol);
          } else if constexpr (is_addv(VAR)) {
            // el from the gathered V row (after the slot loop)
          } else {
            s[t] = ld_node(Qb + uu * qs, pol);
          }
        }
        if constexpr (MODE >= 2) {
  #pragma unroll
          for (int t = 0; t < U; ++t) {
            axpy_n(acc, s[t], vv[t]);
          }
          continue;
        }
        T smax = ninf<T>();
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          if constexpr (MODE == 1) {
            // score read from ES
          } else if constexpr (VAR == GF_DOT) {
            T d, qq;
            if constexpr (GF_FWD_DOT2) {  // paired FFMA2: half the dependent chain
              d = dot_n(qv[t], kv);
              qq = dot_n(qv[t], qv[t]);
            } else {
              d = T(0), qq = T(0);
  #pragma unroll
              for (int i = 0; i < NE; ++i) {
                d += qv[t][i] * kv[i];
                qq += qv[t][i] * qv[t][i];
              }
            }
            d = head_sum(d, lph);
            if (a.l2) d *= inv_norm(head_sum(qq, lph)) * rk;
            s[t] = a.scale * d;
          } else if constexpr (is_addv(VAR)) {
            s[t] = lrelu(head_sum(dot_n(vv[t], al), lph) + erv, a.slope);
          } else {
            s[t] = lrelu(s[t] + erv, a.slope);
          }
          s[t] = ok[t] ? s[t] : ninf<T>();
          smax = GF_FMAX ? fmax(s[t], smax) : (s[t] > smax ? s[t] : smax);
        }
        // Lazy rescale, warp-uniform: only when some lane's running max moves
        // past m + GF_RESCALE_TH.  Below that the stale m is kept: p = e^(s-m)
        // stays <= e^TH, and (m, l) remain a consistent pair (P = e^(s-m) / l
        // for any m), so records, merges and the backward are unchanged.
        if (__any_sync(kFull, smax > m + T(GF_RESCALE_TH))) {
          const T mn = smax > m ? smax : m;
          const T corr = m == mn ? T(1) : expd(m - mn);
          l *= corr;
          scale_n(acc, corr);
          m = mn;
        }
  #pragma unroll
        for (int t = 0; t < U; ++t) {
          const T p = ok[t] ? expd(s[t] - m) : T(0);
          l += p;
          axpy_n(acc, p, vv[t]);
        }
      }
    }
#endif
    if (pk) break;
  }
  if (!pk && eb >= ee) nxt = rsn.y + lane < rsn.z ? ld_idx(a.idx + rsn.y + lane) : 0;

  // Merge the EPW edge slots of the warp (butterfly: every lane ends with
  // the warp's state); packed groups each own a row and skip it.
#pragma unroll
  for (int o = LPE; o < (pk ? LPE : 32); o <<= 1) {
    T acc2[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) acc2[i] = __shfl_xor_sync(kFull, acc[i], o);
    const T m2 = __shfl_xor_sync(kFull, m, o);
    const T l2 = __shfl_xor_sync(kFull, l, o);
    if constexpr (MODE >= 2) {
#pragma unroll
      for (int i = 0; i < NE; ++i) acc[i] += acc2[i];
    } else {
      merge_state<T, NE>(m, l, acc, m2, l2, acc2);
    }
  }

  if (cta) {
    // Shared-memory merge of the 8 warp slices, fixed order w = 0..7.
    __shared__ T sm[kWarpsPerBlock][LPE][2 + NE];
    if (sub == 0) {
      T* d = sm[warp][c];
      d[0] = m;
      d[1] = l;
#pragma unroll
      for (int i = 0; i < NE; ++i) d[2 + i] = acc[i];
    }
    __syncthreads();
    if (warp != 0) return;
    if (sub == 0) {
      const T* d0 = sm[0][c];  // (CTA rows are never packed)
      m = d0[0];
      l = d0[1];
#pragma unroll
      for (int i = 0; i < NE; ++i) acc[i] = d0[2 + i];
      for (int w = 1; w < kWarpsPerBlock; ++w) {
        const T* d = sm[w][c];
        T acc2[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) acc2[i] = d[2 + i];
        if constexpr (MODE >= 2) {
#pragma unroll
          for (int i = 0; i < NE; ++i) acc[i] += acc2[i];
        } else {
          merge_state<T, NE>(m, l, acc, d[0], d[1], acc2);
        }
      }
    }
    if (ct.z > 1) {  // split row: publish this slice; the last CTA merges all slices
      T st[2 + NE];
      st[0] = m;
      st[1] = l;
#pragma unroll
      for (int i = 0; i < NE; ++i) st[2 + i] = acc[i];
      if (!split_publish<2 + NE>(a.part, a.part_cnt, ct, c, LPE, st, sub == 0)) return;
      m = ninf<T>();
      l = T(0);
#pragma unroll
      for (int i = 0; i < NE; ++i) acc[i] = T(0);
      for (int k = 0; k < ct.z; ++k) {
        split_load<2 + NE>(a.part, ct, k, c, LPE, st);
        T acc2[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) acc2[i] = st[2 + i];
        if constexpr (MODE >= 2) {
#pragma unroll
          for (int i = 0; i < NE; ++i) acc[i] += acc2[i];
        } else {
          merge_state<T, NE>(m, l, acc, st[0], st[1], acc2);
        }
      }
    }
  }

  if (pk ? live : sub == 0) {
    const T r = MODE >= 2 ? a.scale : (l == T(0) ? T(0) : T(1) / l);
    T o[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) o[i] = acc[i] * r;
    T* orow = a.O + static_cast<size_t>(v) * a.F + off;
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      st_chunk<T, CB>(orow + k * CW, *reinterpret_cast<T(*)[CW]>(o + k * CW));
    if (MODE < 2 && c % lph == 0) {
      T* rec = a.stats + 4 * (static_cast<size_t>(v) * a.H + h);
      rec[0] = l == T(0) ? ninf<T>() : m;
      rec[1] = l == T(0) ? T(0) : lg2(l);
      rec[2] = VAR == GF_DOT ? rk : erv;
    }
  }
  rs = rsn;
  rsn = rsnn;
  }  // rows
}

// Three buckets (degree-descending order): CTA rows (edge-split over 8
// warps), warp rows, and packed rows (degree <= kSmallDegree, EPW rows per
// warp, one LPE-lane group each); the bucket is warp-uniform.
template <typename T, int CB, int LPE, int CPL, int VAR, int MODE = 0>
__global__ void __launch_bounds__(256, CPL == 1 ? (VAR == GF_ADDV_HBM ? GF_MINB_FWD_H : VAR == GF_ADDV ? GF_MINB_FWD_V : GF_MINB_FWD) : GF_MINB2) fwd_fast(const FwdArgs<T> a) {
  pdl_launch();
  if (a.pf_len[0] > 0) l2_prefetch_tables(a.pf_ptr, a.pf_len);
  pdl_wait();
  constexpr int EPW = 32 / LPE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cb = a.cta_tab ? a.cta_blocks : a.n_cta;  // CTA-bucket blocks
  const int4 one = make_int4(0, 0, 1, -1);
  if (blockIdx.x < static_cast<unsigned>(cb)) {
    const int4 ct = a.cta_tab ? __ldg(a.cta_tab + blockIdx.x) : make_int4(blockIdx.x, 0, 1, -1);
    fwd_row<T, CB, LPE, CPL, VAR, MODE, false>(a, lane, warp, true, ct.x, true, 1, ct);
  } else if (blockIdx.x < static_cast<unsigned>(cb + a.wblocks)) {
    const int slot = a.n_cta + ((blockIdx.x - cb) * kWarpsPerBlock + warp) * a.rpw;
    if (slot >= a.pk0) return;
    if (GF_FWD_LPH1 && CPL == 1 && (is_addv(VAR) || (GF_FWD_LPH1_TABLE && VAR == GF_ADD)) && a.LPH == 1)
      fwd_row<T, CB, LPE, CPL, VAR, MODE, false, 1>(a, lane, warp, false, slot, true,
                                                    min(a.rpw, a.pk0 - slot), one);
    else
      fwd_row<T, CB, LPE, CPL, VAR, MODE, false>(a, lane, warp, false, slot, true,
                                                 min(a.rpw, a.pk0 - slot), one);
  } else if constexpr (EPW > 1) {
    const int slot = a.pk0 + ((blockIdx.x - cb - a.wblocks) * kWarpsPerBlock + warp) * EPW +
                     lane / LPE;
    const bool live = slot < a.n;
    if (!__any_sync(kFull, live)) return;
    fwd_row<T, CB, LPE, CPL, VAR, MODE, true>(a, lane, warp, false, slot, live, 1, one);
  }
}

// ----------------------------------------------------------- generic path --
// Any (H <= 32, D): warp per row, two passes (max, then exp/sum/aggregate),
// per-head scalars owned by lane h, feature accumulators in shared memory.
// Used for shapes whose head does not tile into 16-byte chunks (e.g. D = 5).
template <typename T, int VAR, int MODE = 0>
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
    if constexpr (VAR == GF_DOT && MODE < 2) kvs[f] = __ldg(a.K + static_cast<size_t>(v) * a.F + f);
    acc[f] = T(0);
  }
  __syncwarp();
  T erh = T(0), rkh = T(1);
  if (MODE < 2) generic_row_setup<T, VAR>(a, v, lane, VAR == GF_DOT ? kvs : nullptr, erh, rkh);
  T m = ninf<T>(), l = T(0);
  if (MODE < 2) {
    for (int i = eb; i < ee; ++i) {
      if (lane < a.H) {
        const T s = MODE == 1 ? ld_edge(a.ES + static_cast<size_t>(i) * a.H + lane)
                              : generic_score<T, VAR>(a, __ldg(a.idx + i), v, lane, kvs, erh, rkh);
        m = (m < s || i == eb) ? s : m;  // left-to-right max from the first edge
      }
    }
  }
  for (int i = eb; i < ee; ++i) {
    const int u = __ldg(a.idx + i);
    if (lane < a.H) {
      T p;
      if constexpr (MODE == 3)
        p = ld_edge(a.ES + static_cast<size_t>(__ldg(a.eperm + i)) * a.H + lane);
      else if constexpr (MODE == 2)
        p = ld_edge(a.ES + static_cast<size_t>(i) * a.H + lane);
      else if constexpr (MODE == 1)
        p = expd(ld_edge(a.ES + static_cast<size_t>(i) * a.H + lane) - m);
      else
        p = expd(generic_score<T, VAR>(a, u, v, lane, kvs, erh, rkh) - m);
      l += p;
      ph[lane] = p;
    }
    __syncwarp();
    for (int f = lane; f < a.F; f += 32)
      acc[f] += ph[f / a.D] * __ldg(a.V + static_cast<size_t>(u) * a.F + f);
    __syncwarp();
  }
  if (MODE >= 2) {
    if (lane < a.H) lh[lane] = T(1);
  } else if (lane < a.H) {
    lh[lane] = l;
    T* rec = a.stats + 4 * (static_cast<size_t>(v) * a.H + lane);
    rec[0] = l == T(0) ? ninf<T>() : m;
    rec[1] = l == T(0) ? T(0) : lg2(l);
    rec[2] = VAR == GF_DOT ? rkh : erh;
  }
  __syncwarp();
  for (int f = lane; f < a.F; f += 32) {
    const T lv = lh[f / a.D];
    a.O[static_cast<size_t>(v) * a.F + f] =
        MODE >= 2 ? acc[f] * a.scale : (lv == T(0) ? T(0) : acc[f] / lv);
  }
}

// P materialisation (reference ForwardContext::P, engine.hpp:29): recompute
// p = exp(s - m - log l) per edge and head.  Only on explicit request.
template <typename T, int VAR>
// Warp per row; the per-head row operands (er | 1/||K||, the softmax record)
// are staged in shared memory by lanes h < H, then all 32 lanes stride over
// the row's (edge, head) pairs, so the E x H writes are coalesced and a
// single-head call (the reference API is single-head) keeps every lane busy.
__global__ void __launch_bounds__(128) materialize_p(const FwdArgs<T> a, T* __restrict__ P) {
  __shared__ T s_er[kGenericWarps][32], s_rk[kGenericWarps][32];
  __shared__ Rec<T> s_rec[kGenericWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int v = blockIdx.x * kGenericWarps + warp;
  if (v >= a.n) return;  // warp-uniform
  const int eb = __ldg(a.ptr + v), ee = __ldg(a.ptr + v + 1);
  if (lane < a.H) {
    T erh, rkh;
    generic_row_setup<T, VAR>(a, v, lane, nullptr, erh, rkh);
    s_er[warp][lane] = erh;
    s_rk[warp][lane] = rkh;
    s_rec[warp][lane] = ld_rec(a.stats, static_cast<size_t>(v) * a.H + lane);
  }
  __syncwarp();
  const int total = (ee - eb) * a.H;
  for (int k = lane; k < total; k += 32) {
    const int i = eb + k / a.H, h = k % a.H;
    const int u = __ldg(a.idx + i);
    P[static_cast<size_t>(i) * a.H + h] =
        prob(generic_score<T, VAR>(a, u, v, h, nullptr, s_er[warp][h], s_rk[warp][h]),
             s_rec[warp][h]);
  }
}

template <typename T, int CB, int LPE, int CPL>
int launch_fast_fwd(const FwdArgs<T>& a, int variant, int mode, int blocks, cudaStream_t s) {
  if (mode == 2)  // edge weights given: the score variant is irrelevant
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADD, 2>, blocks, 256, s, a));
  else if (mode == 3)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADD, 3>, blocks, 256, s, a));
  else if (mode == 1 && variant == GF_DOT)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_DOT, 1>, blocks, 256, s, a));
  else if (mode == 1)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADD, 1>, blocks, 256, s, a));
  else if (variant == GF_DOT)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_DOT>, blocks, 256, s, a));
  else if (variant == GF_ADDV)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADDV>, blocks, 256, s, a));
  else if (variant == GF_ADDV_HBM)
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADDV_HBM>, blocks, 256, s, a));
  else
    GF_CHECK_CUDA(launch_k(fwd_fast<T, CB, LPE, CPL, GF_ADD>, blocks, 256, s, a));
  GF_CHECK_LAUNCH("fwd_fast");
  return GF_OK;
}

}  // namespace

#ifdef GF_FWD_PRIMARY  // non-template definitions: emitted by the f32 unit only
FastShape fast_shape(int H, int D, int elem_bytes, int64_t edges) {
  static const int force_cpl = [] {
    const char* e = std::getenv("GF_CPL");
    return e && *e ? std::atoi(e) : 0;
  }();
  FastShape f;
  if (H < 1 || D < 1) return f;
  const long row = static_cast<long>(D) * elem_bytes;
  const int cb = row % 32 == 0 ? 32 : (row % 16 == 0 ? 16 : 0);
  if (!cb) return f;
  const long cph = row / cb;
  auto pow2 = [](long x) { return x > 0 && (x & (x - 1)) == 0; };
  int cpl = cph >= 2 ? 2 : 1;
  if (cpl == 2 && cb == 32 && static_cast<long>(H) * cph <= 32 && force_cpl == 1) cpl = 1;
  (void)edges;
  if (cb == 16 && cpl != 1) return f;  // 16 B chunks only for one-chunk heads
  const long lph = cph / cpl;
  const long lpe = static_cast<long>(H) * lph;
  if (!pow2(cph) || !pow2(lpe) || lpe > 32) return f;
  f.ok = true;
  f.cb = cb;
  f.cpl = cpl;
  f.lph = static_cast<int>(lph);
  f.lpe = static_cast<int>(lpe);
  return f;
}

#endif  // GF_FWD_PRIMARY

static bool aligned(const void* p, int b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; }

template <typename T>
int launch_fwd(const DevGraph& g, const FwdArgs<T>& a0, int variant, cudaStream_t s) {
  return launch_fwd_mode<T>(g, a0, variant, 0, s);
}

template <typename T, int VAR, int MODE>
int launch_generic(const FwdArgs<T>& a, size_t smem, cudaStream_t s) {
  if (smem > 48 * 1024)
    GF_CHECK_CUDA(cudaFuncSetAttribute(fwd_generic<T, VAR, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  const int blocks = (a.n + kGenericWarps - 1) / kGenericWarps;
  fwd_generic<T, VAR, MODE><<<blocks, 32 * kGenericWarps, smem, s>>>(a);
  GF_CHECK_LAUNCH("fwd_generic");
  return GF_OK;
}

template <typename T>
int launch_fwd_mode(const DevGraph& g, const FwdArgs<T>& a0, int variant, int mode,
                    cudaStream_t s) {
  if (g.n == 0) return GF_OK;
  FwdArgs<T> a = a0;
  if (a.n == 0) return GF_OK;  // every row skipped (row-sharded graph)
  const FastShape fs = fast_shape(a.H, a.D, sizeof(T), a.e);
  const bool small = static_cast<int64_t>(g.n) * a.F < (int64_t(1) << 31);  // 32-bit row offsets
  const bool al = fs.ok && small && aligned(a.V, fs.cb) && aligned(a.O, 16) &&
                  aligned(a.stats, 32) &&
                  (mode >= 2 || variant == GF_ADD ||
                   (variant == GF_ADDV && aligned(a.Q, fs.cb) && aligned(a.K, fs.cb)) ||
                   (variant == GF_DOT && aligned(a.Q, fs.cb) && aligned(a.K, 16)));
  if (variant == GF_ADDV && (!al || mode != 0)) {
    set_error("gf_attn_fwd: logits-from-V needs the fast path (callers fall back to el/er tables)");
    return GF_ERR_INVALID;
  }
  // layer form with the gathered V table far beyond L2 (HBM-bound, C5): the
  // high-occupancy instantiation (profiles/r2/ab_r2_gat_layer_form.txt)
  if (variant == GF_ADDV &&
      static_cast<int64_t>(g.n) * a.F * static_cast<int64_t>(sizeof(T)) > (int64_t(100) << 20))
    variant = GF_ADDV_HBM;
  if (al) {
    a.LPH = fs.lph;
    const int epw = 32 / fs.lpe;
    // packed bucket: the small rows (and, unless skipped, the empty ones) when
    // a warp holds more than one edge slot
    a.pk0 = epw > 1 ? std::max(a.n_cta, g.n - a.n_empty - a.n_small) : a.n;
    a.pk0 = std::min(a.pk0, a.n);
    // Short rows (average degree <= 64, e.g. ogbn-products ~26) are latency-
    // bound on their prologue: give each warp 8 consecutive rows and pipeline
    // them; long rows (Reddit ~490) keep one row per warp (A/B, profiles/).
    a.rpw = GF_ROWPIPE ? rows_per_warp(a.e, g.n, a.pk0 - a.n_cta) : 1;
    a.wblocks = (a.pk0 - a.n_cta + kWarpsPerBlock * a.rpw - 1) / (kWarpsPerBlock * a.rpw);
    const int rows_per_block = kWarpsPerBlock * epw;
    const int cta_blocks = a.cta_tab ? a.cta_blocks : a.n_cta;
    const int blocks = cta_blocks + a.wblocks + (a.n - a.pk0 + rows_per_block - 1) / rows_per_block;
    if (l2_prefetch_enabled() && a.e < kPrefetchMaxEdges && mode <= 1) {
      // the gathered tables: V, and Q (dot) | el (table-form GAT)
      const int64_t vb = static_cast<int64_t>(g.n) * a.F * static_cast<int64_t>(sizeof(T));
      const int64_t qb = variant == GF_DOT ? vb
                         : is_addv(variant) ? 0
                                            : static_cast<int64_t>(g.n) * a.H * sizeof(T);
      if (vb + qb <= kPrefetchMaxBytes) {
        a.pf_ptr[0] = a.V, a.pf_len[0] = vb;
        a.pf_ptr[1] = a.Q, a.pf_len[1] = qb;
      }
    }
    // split super rows: slice states + arrival counters (stream-ordered scratch)
    if (a.cta_tab && a.parts > 0) {
      const size_t nv = 2 + static_cast<size_t>(fs.cpl) * (fs.cb / sizeof(T));
      GF_CHECK_CUDA(scratch_alloc(&a.part, sizeof(T) * a.parts * fs.lpe * nv, s));
      GF_CHECK_CUDA(scratch_alloc(&a.part_cnt, sizeof(unsigned) * a.parts, s));
      GF_CHECK_CUDA(cudaMemsetAsync(a.part_cnt, 0, sizeof(unsigned) * a.parts, s));
    }
    struct PartFree {
      FwdArgs<T>& a;
      cudaStream_t s;
      ~PartFree() {
        if (a.part) cudaFreeAsync(a.part, s);
        if (a.part_cnt) cudaFreeAsync(a.part_cnt, s);
      }
    } part_free{a, s};
    const int key = fs.cb * 1000 + fs.lpe * 10 + fs.cpl;
    switch (key) {
      case 32011: return launch_fast_fwd<T, 32, 1, 1>(a, variant, mode, blocks, s);
      case 32021: return launch_fast_fwd<T, 32, 2, 1>(a, variant, mode, blocks, s);
      case 32041: return launch_fast_fwd<T, 32, 4, 1>(a, variant, mode, blocks, s);
      case 32081: return launch_fast_fwd<T, 32, 8, 1>(a, variant, mode, blocks, s);
      case 32161: return launch_fast_fwd<T, 32, 16, 1>(a, variant, mode, blocks, s);
      case 32321: return launch_fast_fwd<T, 32, 32, 1>(a, variant, mode, blocks, s);
      case 32012: return launch_fast_fwd<T, 32, 1, 2>(a, variant, mode, blocks, s);
      case 32022: return launch_fast_fwd<T, 32, 2, 2>(a, variant, mode, blocks, s);
      case 32042: return launch_fast_fwd<T, 32, 4, 2>(a, variant, mode, blocks, s);
      case 32082: return launch_fast_fwd<T, 32, 8, 2>(a, variant, mode, blocks, s);
      case 32162: return launch_fast_fwd<T, 32, 16, 2>(a, variant, mode, blocks, s);
      case 32322: return launch_fast_fwd<T, 32, 32, 2>(a, variant, mode, blocks, s);
      case 16011: return launch_fast_fwd<T, 16, 1, 1>(a, variant, mode, blocks, s);
      case 16021: return launch_fast_fwd<T, 16, 2, 1>(a, variant, mode, blocks, s);
      case 16041: return launch_fast_fwd<T, 16, 4, 1>(a, variant, mode, blocks, s);
      case 16081: return launch_fast_fwd<T, 16, 8, 1>(a, variant, mode, blocks, s);
      case 16161: return launch_fast_fwd<T, 16, 16, 1>(a, variant, mode, blocks, s);
      case 16321: return launch_fast_fwd<T, 16, 32, 1>(a, variant, mode, blocks, s);
      default: break;
    }
  }
  if (a.H > 32) {
    set_error("gf_attn_fwd: heads > 32 need a head shape that tiles into 16/32-byte chunks");
    return GF_ERR_UNSUPPORTED;
  }
  const size_t smem = static_cast<size_t>(kGenericWarps) * (2 * a.F + 64) * sizeof(T);
  if (smem > 200 * 1024) {
    set_error("gf_attn_fwd: feature width too large for the generic path");
    return GF_ERR_UNSUPPORTED;
  }
  if (mode == 2) return launch_generic<T, GF_ADD, 2>(a, smem, s);
  if (mode == 3) return launch_generic<T, GF_ADD, 3>(a, smem, s);
  if (mode == 1)
    return variant == GF_DOT ? launch_generic<T, GF_DOT, 1>(a, smem, s)
                             : launch_generic<T, GF_ADD, 1>(a, smem, s);
  return variant == GF_DOT ? launch_generic<T, GF_DOT, 0>(a, smem, s)
                           : launch_generic<T, GF_ADD, 0>(a, smem, s);
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

}  // namespace gfb

// Drop-in operator API over the B200 C-ABI: run_strategy & variants
// (engine.hpp:233-336), fused/unfused_backward (autograd.hpp:196-226),
// finite_difference_check (autograd.hpp:241-287), matmul / conv_forward /
// conv_backward / make_pipeline_inputs (models.hpp:58-190).
//
// Every compute step is a gf_* call into libgraphfuse_cuda.so; this file only
// validates arguments exactly like the reference (same exception types and
// message prefixes), moves host vectors to/from HBM and keeps the reference's
// modelled counters.  No CPU compute fallback exists.
#include <chrono>
#include <algorithm>
#include <limits>
#include <mutex>

#include "gf_cuda.h"
#include "graphfuse/graphfuse.hpp"

namespace graphfuse {

namespace detail {

[[noreturn]] void device_fail(const char* what) {
  throw EngineError(std::string("B200 path: ") + what + ": " + gf_last_error());
}

void need_device() {
  static const bool ok = gf_device_ok() != 0;
  if (!ok)
    throw EngineError(
        "B200 path: no sm_100 device available (libgraphfuse_cuda has no CPU fallback)");
}

#define GFH_CALL(expr)                     \
  do {                                     \
    if ((expr) != GF_OK) ::graphfuse::detail::device_fail(#expr); \
  } while (0)

/// Owning device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) : bytes(b) { GFH_CALL(gf_malloc(b, &p)); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  ~DevBuf() { gf_free(p); }
  template <typename T>
  static DevBuf from(const std::vector<T>& h) {
    DevBuf d(sizeof(T) * h.size());
    if (!h.empty()) GFH_CALL(gf_memcpy(d.p, h.data(), d.bytes, 0, nullptr));
    return d;
  }
  template <typename T>
  void to(std::vector<T>& h) const {
    if (!h.empty()) GFH_CALL(gf_memcpy(h.data(), p, sizeof(T) * h.size(), 1, nullptr));
  }
};

struct DeviceGraphCache {
  gf_graph_t h = nullptr;
  NodeId n = -1;
  EdgeId e = -1;
  const void* row_data = nullptr;
  const void* col_data = nullptr;
  const void* csc_ptr_data = nullptr;
  const void* csc_row_data = nullptr;
  std::int64_t thr = 0;
  ~DeviceGraphCache() {
    if (h) gf_graph_destroy(h);
  }
};

// The device copy is keyed on the Graph's sizes, the addresses of all four
// topology arrays and the CTA threshold.  Like the reference's Graph (SPEC:
// immutable, shareable), a Graph must not be edited in place after its first
// device call; concurrent callers on one Graph are serialised by the mutex
// while the cache is checked or rebuilt.
gf_graph_t device_graph(const Graph& g, const FusionPlan& plan) {
  need_device();
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto& c = g.device;
  if (!c || c->n != g.num_nodes || c->e != g.num_edges ||
      c->row_data != g.csr_row_ptr.data() || c->col_data != g.csr_col_idx.data() ||
      c->csc_ptr_data != g.csc_col_ptr.data() || c->csc_row_data != g.csc_row_idx.data() ||
      c->thr != plan.cta_row_threshold) {
    auto fresh = std::make_shared<DeviceGraphCache>();
    GFH_CALL(gf_graph_create(g.num_nodes, g.num_edges, g.csr_row_ptr.data(),
                             g.csr_col_idx.data(), g.csc_col_ptr.data(), g.csc_row_idx.data(),
                             static_cast<std::int32_t>(plan.cta_row_threshold), nullptr,
                             &fresh->h));
    fresh->n = g.num_nodes;
    fresh->e = g.num_edges;
    fresh->row_data = g.csr_row_ptr.data();
    fresh->col_data = g.csr_col_idx.data();
    fresh->csc_ptr_data = g.csc_col_ptr.data();
    fresh->csc_row_data = g.csc_row_idx.data();
    fresh->thr = plan.cta_row_threshold;
    c = std::move(fresh);
  }
  return c->h;
}

template <typename T>
constexpr int dtype_code() {
  return sizeof(T) == 8 ? GF_F64 : GF_F32;
}

template <typename T>
gf_attn_desc make_desc(const SddmmKind& kind, std::int64_t d) {
  gf_attn_desc a{};
  a.dtype = dtype_code<T>();
  a.variant = kind.variant == SddmmVariant::Add ? GF_ADD : GF_DOT;
  a.l2 = kind.variant == SddmmVariant::Dot && kind.l2_normalize_inputs ? 1 : 0;
  a.heads = 1;
  a.head_dim = static_cast<std::int32_t>(d);
  a.scale = kind.scale;
  a.slope = kind.leaky_slope;
  return a;
}

template <typename T>
void validate_inputs(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                     const DenseMatrix<T>& V, const SddmmKind& kind) {
  if (V.rows != g.num_nodes) throw KernelError("engine: V.rows must equal N");
  if (kind.variant == SddmmVariant::Dot &&
      (Q.rows != g.num_nodes || K.rows != g.num_nodes || Q.cols != K.cols))
    throw KernelError("engine: Q/K dimension mismatch");
  if (kind.variant == SddmmVariant::Add && (Q.cols != 1 || K.cols != 1))
    throw KernelError("engine: add-SDDMM expects N x 1 el/er");
  if (kind.variant == SddmmVariant::Add && (Q.rows != g.num_nodes || K.rows != g.num_nodes))
    throw KernelError("engine: el/er must have N rows");
}

/// Dot attention whose Q/K width differs from V's (the reference allows it,
/// engine.hpp:239-243): the fused kernels take one head width, so these run
/// the device's unfused single-step schedule (SDDMM -> softmax -> SpMM; the
/// 5-launch unfused backward) instead.
template <typename T>
bool split_width(const DenseMatrix<T>& Q, const DenseMatrix<T>& V, const SddmmKind& kind) {
  return kind.variant == SddmmVariant::Dot && Q.cols != V.cols;
}

int strategy_code(Strategy s) {
  switch (s) {
    case Strategy::Pmf: return GF_STRAT_PMF;
    case Strategy::Unfused: return GF_STRAT_UNFUSED;
    case Strategy::FeatureParallelBaseline: return GF_STRAT_BASELINE;
    default: return GF_STRAT_SMMF;
  }
}

/// Device forward under `mode`'s kernels: returns O and lse (and P when want_p).
template <typename T>
void device_forward(const Graph& g, const FusionPlan& plan, const DenseMatrix<T>& Q,
                    const DenseMatrix<T>& K, const DenseMatrix<T>& V, const SddmmKind& kind,
                    std::vector<T>& O, std::vector<T>& lse, std::vector<T>* P,
                    Strategy mode = Strategy::Smmf) {
  gf_graph_t dg = device_graph(g, plan);
  const std::int64_t d = V.cols;
  const gf_attn_desc desc = make_desc<T>(kind, d);
  DevBuf dq = DevBuf::from(Q.data), dk = DevBuf::from(K.data), dv = DevBuf::from(V.data);
  O.assign(static_cast<size_t>(g.num_nodes * d), T(0));
  if (split_width(Q, V, kind)) {  // unfused device schedule over two head widths
    lse.clear();  // no softmax records: the backward takes the unfused schedule too
    const gf_attn_desc qd = make_desc<T>(kind, Q.cols);
    const size_t eb = sizeof(T) * static_cast<size_t>(std::max<EdgeId>(g.num_edges, 1));
    DevBuf ds(eb), dp(eb), dO(sizeof(T) * std::max<size_t>(O.size(), 1));
    if (g.num_edges > 0 && Q.cols > 0) GFH_CALL(gf_sddmm(dg, &qd, dq.p, dk.p, ds.p, nullptr));
    else GFH_CALL(gf_memset(ds.p, 0, eb, nullptr));
    GFH_CALL(gf_edge_softmax(dg, desc.dtype, 1, ds.p, dp.p, nullptr));
    if (d > 0)
      GFH_CALL(gf_spmm(dg, desc.dtype, 1, static_cast<std::int32_t>(d), dp.p, dv.p, dO.p, nullptr));
    GFH_CALL(gf_stream_sync(nullptr));
    if (d > 0) dO.to(O);
    if (P) {
      P->assign(static_cast<size_t>(g.num_edges), T(0));
      dp.to(*P);
    }
    return;
  }
  lse.assign(static_cast<size_t>(4 * g.num_nodes), T(0));  // softmax records (4 per row)
  DevBuf dO(sizeof(T) * O.size()), dl(sizeof(T) * lse.size());
  DevBuf dp(P ? sizeof(T) * static_cast<size_t>(g.num_edges) : 0);
  GFH_CALL(gf_attn_fwd_strategy(dg, &desc, strategy_code(mode), dq.p, dk.p, dv.p, dO.p, dl.p,
                                P ? dp.p : nullptr, nullptr, 0, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  dO.to(O);
  dl.to(lse);
  if (P) {
    P->assign(static_cast<size_t>(g.num_edges), T(0));
    dp.to(*P);
  }
}

/// Measured GPU time (ms) of `mode`'s forward kernels on device-resident
/// copies of Q, K, V (the bench harness's measured column).
template <typename T>
double device_forward_ms(const Graph& g, const FusionPlan& plan, const DenseMatrix<T>& Q,
                         const DenseMatrix<T>& K, const DenseMatrix<T>& V, const SddmmKind& kind,
                         Strategy mode, int reps) {
  validate_inputs(g, Q, K, V, kind);
  gf_graph_t dg = device_graph(g, plan);
  const gf_attn_desc desc = make_desc<T>(kind, V.cols);
  DevBuf dq = DevBuf::from(Q.data), dk = DevBuf::from(K.data), dv = DevBuf::from(V.data);
  DevBuf dO(sizeof(T) * static_cast<size_t>(g.num_nodes * V.cols)),
      dl(sizeof(T) * static_cast<size_t>(4 * g.num_nodes));
  float ms = 0.f;
  GFH_CALL(gf_time_fwd_strategy(dg, &desc, strategy_code(mode), dq.p, dk.p, dv.p, dO.p, dl.p,
                                reps, &ms, nullptr));
  return ms;
}
/// Measured DRAM bytes (read + write, CUPTI range profiler through
/// gf_measure_metrics) of `mode`'s forward kernels on device-resident inputs,
/// L2 flushed (256 MiB write) before the profiled range.  Returns -1 when the
/// counters are unavailable (no libcupti / no profiling permission).
template <typename T>
double device_forward_dram_bytes(const Graph& g, const FusionPlan& plan, const DenseMatrix<T>& Q,
                                 const DenseMatrix<T>& K, const DenseMatrix<T>& V,
                                 const SddmmKind& kind, Strategy mode) {
  validate_inputs(g, Q, K, V, kind);
  struct Region {
    gf_graph_t dg;
    gf_attn_desc desc;
    int strategy;
    void *q, *k, *v, *o, *l, *flush;
    size_t flush_bytes;
  };
  DevBuf dq = DevBuf::from(Q.data), dk = DevBuf::from(K.data), dv = DevBuf::from(V.data);
  DevBuf dO(sizeof(T) * static_cast<size_t>(std::max<std::int64_t>(1, g.num_nodes * V.cols))),
      dl(sizeof(T) * static_cast<size_t>(std::max<std::int64_t>(1, 4 * g.num_nodes)));
  const size_t fb = size_t(256) << 20;
  DevBuf flush(fb);
  Region r{device_graph(g, plan), make_desc<T>(kind, V.cols), strategy_code(mode), dq.p, dk.p,
           dv.p, dO.p, dl.p, flush.p, fb};
  auto prep = [](void* u) {
    auto* x = static_cast<Region*>(u);
    gf_l2_reset_persisting();
    gf_memset(x->flush, 0, x->flush_bytes, nullptr);
  };
  auto run = [](void* u) {
    auto* x = static_cast<Region*>(u);
    gf_attn_fwd_strategy(x->dg, &x->desc, x->strategy, x->q, x->k, x->v, x->o, x->l, nullptr,
                         nullptr, 0, nullptr);
  };
  const char* names[2] = {"dram__bytes_read.sum", "dram__bytes_write.sum"};
  double vals[2] = {0, 0};
  // A counter session can fail transiently (e.g. the profiler being busy):
  // retry once, and report the column as unavailable rather than failing the
  // benchmark over a diagnostic.
  int rc = gf_measure_metrics(prep, run, &r, names, 2, vals);
  if (rc != GF_OK && rc != GF_ERR_UNSUPPORTED) rc = gf_measure_metrics(prep, run, &r, names, 2, vals);
  if (rc != GF_OK) return -1.0;
  return vals[0] + vals[1];
}
template double device_forward_dram_bytes<float>(const Graph&, const FusionPlan&,
                                                 const DenseMatrix<float>&,
                                                 const DenseMatrix<float>&,
                                                 const DenseMatrix<float>&, const SddmmKind&,
                                                 Strategy);
template double device_forward_dram_bytes<double>(const Graph&, const FusionPlan&,
                                                  const DenseMatrix<double>&,
                                                  const DenseMatrix<double>&,
                                                  const DenseMatrix<double>&, const SddmmKind&,
                                                  Strategy);
template double device_forward_ms<float>(const Graph&, const FusionPlan&, const DenseMatrix<float>&,
                                         const DenseMatrix<float>&, const DenseMatrix<float>&,
                                         const SddmmKind&, Strategy, int);
template double device_forward_ms<double>(const Graph&, const FusionPlan&,
                                          const DenseMatrix<double>&, const DenseMatrix<double>&,
                                          const DenseMatrix<double>&, const SddmmKind&, Strategy,
                                          int);

template <typename T>
ForwardResult<T> run_mode(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                          const DenseMatrix<T>& V, const SddmmKind& kind, const FusionPlan& plan,
                          Strategy mode) {
  validate_inputs(g, Q, K, V, kind);
  const std::int64_t d = V.cols;
  if (mode == Strategy::Smmf) check_smmf_feasible<T>(g, plan, d);
  const auto t0 = std::chrono::steady_clock::now();
  ForwardResult<T> res;
  res.ctx.g = &g;
  res.ctx.Q = Q;
  res.ctx.K = K;
  res.ctx.V = V;
  res.ctx.kind = kind;
  res.ctx.plan = plan.with_strategy(mode);
  device_forward(g, plan, Q, K, V, kind, res.ctx.O, res.ctx.lse, &res.ctx.P.values, mode);
  res.O = DenseMatrix<T>(g.num_nodes, d);
  res.O.data = res.ctx.O;
  res.counters = model_counters<T>(g, kind, plan, d, mode);
  res.counters.elapsed_ns = static_cast<std::uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
          .count());
  return res;
}

template ForwardResult<float> run_mode<float>(const Graph&, const DenseMatrix<float>&,
                                              const DenseMatrix<float>&, const DenseMatrix<float>&,
                                              const SddmmKind&, const FusionPlan&, Strategy);
template ForwardResult<double> run_mode<double>(const Graph&, const DenseMatrix<double>&,
                                                const DenseMatrix<double>&,
                                                const DenseMatrix<double>&, const SddmmKind&,
                                                const FusionPlan&, Strategy);

ExecCounters backward_counters(const Graph& g, std::int64_t d, std::uint64_t b,
                               std::uint64_t launches) {
  ExecCounters c;
  const std::uint64_t E = static_cast<std::uint64_t>(g.num_edges);
  const std::uint64_t N = static_cast<std::uint64_t>(g.num_nodes);
  const std::uint64_t dd = static_cast<std::uint64_t>(d);
  c.kernel_launches = launches;
  c.global_bytes_read = 4 * E * dd * b + 2 * E * b;
  c.global_bytes_written = 2 * N * dd * b + 2 * E * b;
  if (launches >= 5) {  // edge gradients round-trip in the unfused schedule
    c.global_bytes_read += 2 * E * b;
    c.global_bytes_written += 2 * E * b;
  }
  return c;
}

template <typename T>
GradBundle<T> backward_values(const Graph& g, const ForwardContext<T>& ctx,
                              const DenseMatrix<T>& dO);

template <typename T>
GradBundle<T> device_backward(const Graph& g, const ForwardContext<T>& ctx,
                              const DenseMatrix<T>& dO) {
  const auto& V = ctx.V;
  if (dO.rows != g.num_nodes || dO.cols != V.cols)
    throw KernelError("spmm_backward: dO shape mismatch");
  validate_inputs(g, ctx.Q, ctx.K, V, ctx.kind);
  if (split_width(ctx.Q, V, ctx.kind)) return backward_values(g, ctx, dO);
  const std::int64_t d = V.cols;
  const FusionPlan& plan = ctx.plan;
  std::vector<T> O = ctx.O, lse = ctx.lse;
  if (O.size() != static_cast<size_t>(g.num_nodes * d) ||
      lse.size() != static_cast<size_t>(4 * g.num_nodes))
    device_forward(g, plan, ctx.Q, ctx.K, V, ctx.kind, O, lse, static_cast<std::vector<T>*>(nullptr));  // hand-built ctx
  gf_graph_t dg = device_graph(g, plan);
  const gf_attn_desc desc = make_desc<T>(ctx.kind, d);
  DevBuf dq = DevBuf::from(ctx.Q.data), dk = DevBuf::from(ctx.K.data),
         dv = DevBuf::from(V.data), dob = DevBuf::from(O), dl = DevBuf::from(lse),
         ddo = DevBuf::from(dO.data);
  GradBundle<T> gb;
  gb.dQ = DenseMatrix<T>(ctx.Q.rows, ctx.Q.cols);
  gb.dK = DenseMatrix<T>(ctx.K.rows, ctx.K.cols);
  gb.dV = DenseMatrix<T>(V.rows, V.cols);
  DevBuf gq(sizeof(T) * gb.dQ.data.size()), gk(sizeof(T) * gb.dK.data.size()),
      gv(sizeof(T) * gb.dV.data.size());
  GFH_CALL(gf_attn_bwd(dg, &desc, dq.p, dk.p, dv.p, dob.p, dl.p, ddo.p, gq.p, gk.p, gv.p,
                       nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  gq.to(gb.dQ.data);
  gk.to(gb.dK.data);
  gv.to(gb.dV.data);
  return gb;
}

}  // namespace detail

// ---------------------------------------------------- single-step ops --
namespace detail {

template <typename T>
gf_attn_desc step_desc(SddmmVariant v, std::int64_t d, double scale, double slope, bool l2) {
  gf_attn_desc a{};
  a.dtype = dtype_code<T>();
  a.variant = v == SddmmVariant::Add ? GF_ADD : GF_DOT;
  a.l2 = l2 ? 1 : 0;
  a.heads = 1;
  a.head_dim = static_cast<std::int32_t>(std::max<std::int64_t>(1, d));
  a.scale = scale;
  a.slope = slope;
  return a;
}

template <typename T>
EdgeScalars<T> sddmm_device(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                            const gf_attn_desc& desc) {
  EdgeScalars<T> s(g.num_edges);
  if (g.num_edges == 0) return s;
  gf_graph_t dg = device_graph(g, FusionPlan{});
  DevBuf dq = DevBuf::from(Q.data), dk = DevBuf::from(K.data), ds(sizeof(T) * s.values.size());
  GFH_CALL(gf_sddmm(dg, &desc, dq.p, dk.p, ds.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  ds.to(s.values);
  return s;
}

template <typename T>
GradBundle<T> backward_values(const Graph& g, const ForwardContext<T>& ctx,
                              const DenseMatrix<T>& dO) {
  const auto& V = ctx.V;
  if (dO.rows != g.num_nodes || dO.cols != V.cols)
    throw KernelError("spmm_backward: dO shape mismatch");
  validate_inputs(g, ctx.Q, ctx.K, V, ctx.kind);
  std::vector<T> P = ctx.P.values;
  if (P.size() != static_cast<size_t>(g.num_edges)) {  // hand-built context: rebuild P
    std::vector<T> O, lse;
    device_forward(g, FusionPlan{}, ctx.Q, ctx.K, V, ctx.kind, O, lse, &P);
  }
  GradBundle<T> gb;
  const std::int64_t d = V.cols, E = g.num_edges;
  gb.dQ = DenseMatrix<T>(ctx.Q.rows, ctx.Q.cols);
  gb.dK = DenseMatrix<T>(ctx.K.rows, ctx.K.cols);
  gb.dV = DenseMatrix<T>(V.rows, d);
  gb.dP = EdgeScalars<T>(E);
  gb.dS = EdgeScalars<T>(E);
  if (g.num_nodes == 0 || d == 0) return gb;
  gf_graph_t dg = device_graph(g, ctx.plan);
  // sddmm_backward works on the Q/K width (== d except for split widths)
  const gf_attn_desc desc =
      make_desc<T>(ctx.kind, ctx.kind.variant == SddmmVariant::Dot ? ctx.Q.cols : d);
  DevBuf dq = DevBuf::from(ctx.Q.data), dk = DevBuf::from(ctx.K.data), dv = DevBuf::from(V.data),
         dp = DevBuf::from(P), ddo = DevBuf::from(dO.data);
  DevBuf gdp(sizeof(T) * std::max<std::int64_t>(E, 1)), gds(sizeof(T) * std::max<std::int64_t>(E, 1));
  DevBuf gq(sizeof(T) * gb.dQ.data.size()), gk(sizeof(T) * gb.dK.data.size()),
      gv(sizeof(T) * gb.dV.data.size());
  const std::int32_t dt = dtype_code<T>(), D = static_cast<std::int32_t>(d);
  // 5 launches: dP (SDDMM), dV (CSC SpMM), dS (softmax bwd), dK (CSR), dQ (CSC)
  GFH_CALL(gf_spmm_backward(dg, dt, 1, D, dp.p, dv.p, ddo.p, gdp.p, gv.p, nullptr));
  GFH_CALL(gf_softmax_backward(dg, dt, 1, dp.p, gdp.p, gds.p, nullptr));
  GFH_CALL(gf_sddmm_backward(dg, &desc, dq.p, dk.p, gds.p, gq.p, gk.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  gq.to(gb.dQ.data);
  gk.to(gb.dK.data);
  gv.to(gb.dV.data);
  gdp.to(gb.dP.values);
  gds.to(gb.dS.values);
  return gb;
}

template <typename T>
ExecCounters backward_counter_model(const Graph& g, const ForwardContext<T>& ctx,
                                    std::int64_t launches) {
  return backward_counters(g, ctx.V.cols, sizeof(T), static_cast<std::uint64_t>(launches));
}

}  // namespace detail

template <typename T>
EdgeScalars<T> sddmm_dot(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                         T scale) {
  if (Q.rows != g.num_nodes || K.rows != g.num_nodes || Q.cols != K.cols)
    throw KernelError("sddmm_dot: dimension mismatch");
  if (Q.cols == 0) return EdgeScalars<T>(g.num_edges);
  return detail::sddmm_device(
      g, Q, K, detail::step_desc<T>(SddmmVariant::Dot, Q.cols, scale, 0.0, false));
}

template <typename T>
EdgeScalars<T> sddmm_add(const Graph& g, const DenseMatrix<T>& el, const DenseMatrix<T>& er,
                         T leaky_slope) {
  if (el.rows != g.num_nodes || er.rows != g.num_nodes || el.cols != 1 || er.cols != 1)
    throw KernelError("sddmm_add: el/er must be N x 1");
  return detail::sddmm_device(
      g, el, er, detail::step_desc<T>(SddmmVariant::Add, 1, 1.0, leaky_slope, false));
}

template <typename T>
DenseMatrix<T> l2_normalize_rows(const DenseMatrix<T>& X, T eps) {
  if (eps <= T(0)) throw KernelError("l2_normalize_rows: eps must be > 0");
  DenseMatrix<T> out(X.rows, X.cols);
  if (X.rows == 0 || X.cols == 0) return out;
  detail::need_device();
  detail::DevBuf x = detail::DevBuf::from(X.data), y(sizeof(T) * out.data.size());
  GFH_CALL(gf_l2_normalize_rows(detail::dtype_code<T>(), X.rows, 1,
                                static_cast<std::int32_t>(X.cols), x.p, y.p, eps, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  y.to(out.data);
  return out;
}

template <typename T>
DenseMatrix<T> l2_normalize_backward(const DenseMatrix<T>& X, const DenseMatrix<T>& dY, T eps) {
  if (dY.rows != X.rows || dY.cols != X.cols)
    throw KernelError("l2_normalize_backward: shape mismatch");
  DenseMatrix<T> dX(X.rows, X.cols);
  if (X.rows == 0 || X.cols == 0) return dX;
  detail::need_device();
  detail::DevBuf x = detail::DevBuf::from(X.data), dy = detail::DevBuf::from(dY.data),
                 dx(sizeof(T) * dX.data.size());
  GFH_CALL(gf_l2_normalize_backward(detail::dtype_code<T>(), X.rows, 1,
                                    static_cast<std::int32_t>(X.cols), x.p, dy.p, dx.p, eps,
                                    nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  dx.to(dX.data);
  return dX;
}

template <typename T>
EdgeScalars<T> edge_softmax(const Graph& g, const EdgeScalars<T>& s) {
  if (s.size() != g.num_edges) throw KernelError("edge_softmax: length mismatch");
  EdgeScalars<T> p(g.num_edges);
  if (g.num_edges == 0) return p;
  gf_graph_t dg = detail::device_graph(g, FusionPlan{});
  detail::DevBuf ds = detail::DevBuf::from(s.values), dp(sizeof(T) * p.values.size());
  GFH_CALL(gf_edge_softmax(dg, detail::dtype_code<T>(), 1, ds.p, dp.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  dp.to(p.values);
  return p;
}

template <typename T>
std::pair<DenseMatrix<T>, DenseMatrix<T>> dense_oracle_forward(const Graph& g,
                                                               const DenseMatrix<T>& Q,
                                                               const DenseMatrix<T>& K,
                                                               const DenseMatrix<T>& V,
                                                               const SddmmKind& kind) {
  if (g.num_nodes > 4096) throw KernelError("dense_oracle_forward: N > 4096");
  const NodeId n = g.num_nodes;
  const std::int64_t qk = kind.variant == SddmmVariant::Dot ? Q.cols : 1;
  if (Q.rows != n || K.rows != n || V.rows != n || K.cols != Q.cols ||
      (kind.variant == SddmmVariant::Add && Q.cols != 1))
    throw KernelError("dense_oracle_forward: dimension mismatch");
  DenseMatrix<T> S(n, n), O(n, V.cols);
  if (n == 0) return {std::move(S), std::move(O)};
  detail::need_device();
  gf_attn_desc d = detail::step_desc<T>(kind.variant, qk, kind.scale, kind.leaky_slope,
                                        kind.variant == SddmmVariant::Dot &&
                                            kind.l2_normalize_inputs);
  detail::DevBuf src = detail::DevBuf::from(g.coo_src), dst = detail::DevBuf::from(g.coo_dst),
                 dq = detail::DevBuf::from(Q.data), dk = detail::DevBuf::from(K.data),
                 dv = detail::DevBuf::from(V.data), ds(sizeof(T) * S.data.size()),
                 dO(sizeof(T) * std::max<size_t>(O.data.size(), 1));
  GFH_CALL(gf_dense_oracle_forward(n, g.num_edges, static_cast<const std::int64_t*>(src.p),
                                   static_cast<const std::int64_t*>(dst.p), &d, V.cols, dq.p,
                                   dk.p, dv.p, ds.p, dO.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  ds.to(S.data);
  dO.to(O.data);
  return {std::move(S), std::move(O)};
}

template <typename T>
DenseMatrix<T> spmm(const Graph& g, const EdgeScalars<T>& p, const DenseMatrix<T>& V) {
  if (V.rows != g.num_nodes) throw KernelError("spmm: V.rows must equal N");
  if (p.size() != g.num_edges) throw KernelError("spmm: P length mismatch");
  DenseMatrix<T> out(g.num_nodes, V.cols);
  if (g.num_nodes == 0 || V.cols == 0) return out;
  gf_graph_t dg = detail::device_graph(g, FusionPlan{});
  detail::DevBuf dp = detail::DevBuf::from(p.values), dv = detail::DevBuf::from(V.data),
                 o(sizeof(T) * out.data.size());
  GFH_CALL(gf_spmm(dg, detail::dtype_code<T>(), 1, static_cast<std::int32_t>(V.cols), dp.p, dv.p,
                   o.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  o.to(out.data);
  return out;
}

template <typename T>
EdgeScalars<T> sddmm(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                     const SddmmKind& kind) {
  if (kind.variant == SddmmVariant::Add)
    return sddmm_add(g, Q, K, static_cast<T>(kind.leaky_slope));
  if (!kind.l2_normalize_inputs) return sddmm_dot(g, Q, K, static_cast<T>(kind.scale));
  if (Q.rows != g.num_nodes || K.rows != g.num_nodes || Q.cols != K.cols)
    throw KernelError("sddmm_dot: dimension mismatch");
  if (Q.cols == 0) return EdgeScalars<T>(g.num_edges);
  return detail::sddmm_device(
      g, Q, K, detail::step_desc<T>(SddmmVariant::Dot, Q.cols, kind.scale, 0.0, true));
}

template <typename T>
std::pair<EdgeScalars<T>, DenseMatrix<T>> spmm_backward(const Graph& g, const EdgeScalars<T>& P,
                                                        const DenseMatrix<T>& V,
                                                        const DenseMatrix<T>& dO) {
  if (dO.rows != g.num_nodes || dO.cols != V.cols)
    throw KernelError("spmm_backward: dO shape mismatch");
  if (V.rows != g.num_nodes || P.size() != g.num_edges)
    throw KernelError("spmm_backward: P / V shape mismatch");
  EdgeScalars<T> dP(g.num_edges);
  DenseMatrix<T> dV(g.num_nodes, V.cols);
  if (g.num_nodes == 0 || V.cols == 0) return {std::move(dP), std::move(dV)};
  gf_graph_t dg = detail::device_graph(g, FusionPlan{});
  detail::DevBuf dp = detail::DevBuf::from(P.values), dv = detail::DevBuf::from(V.data),
                 ddo = detail::DevBuf::from(dO.data),
                 gdp(sizeof(T) * std::max<std::int64_t>(g.num_edges, 1)),
                 gv(sizeof(T) * dV.data.size());
  GFH_CALL(gf_spmm_backward(dg, detail::dtype_code<T>(), 1, static_cast<std::int32_t>(V.cols),
                            dp.p, dv.p, ddo.p, gdp.p, gv.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  gdp.to(dP.values);
  gv.to(dV.data);
  return {std::move(dP), std::move(dV)};
}

template <typename T>
EdgeScalars<T> softmax_backward(const Graph& g, const EdgeScalars<T>& P, const EdgeScalars<T>& dP) {
  if (P.size() != g.num_edges || dP.size() != g.num_edges)
    throw KernelError("softmax_backward: length mismatch");
  EdgeScalars<T> dS(g.num_edges);
  if (g.num_edges == 0) return dS;
  gf_graph_t dg = detail::device_graph(g, FusionPlan{});
  detail::DevBuf p = detail::DevBuf::from(P.values), dp = detail::DevBuf::from(dP.values),
                 ds(sizeof(T) * dS.values.size());
  GFH_CALL(gf_softmax_backward(dg, detail::dtype_code<T>(), 1, p.p, dp.p, ds.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  ds.to(dS.values);
  return dS;
}

template <typename T>
std::pair<DenseMatrix<T>, DenseMatrix<T>> sddmm_backward(const Graph& g, const DenseMatrix<T>& Q,
                                                         const DenseMatrix<T>& K,
                                                         const EdgeScalars<T>& dS,
                                                         const SddmmKind& kind) {
  if (dS.size() != g.num_edges) throw KernelError("sddmm_backward: dS length mismatch");
  const bool add = kind.variant == SddmmVariant::Add;
  if (add ? (Q.rows != g.num_nodes || K.rows != g.num_nodes || Q.cols != 1 || K.cols != 1)
          : (Q.rows != g.num_nodes || K.rows != g.num_nodes || Q.cols != K.cols))
    throw KernelError("sddmm_backward: Q/K shape mismatch");
  DenseMatrix<T> dQ(g.num_nodes, Q.cols), dK(g.num_nodes, K.cols);
  if (g.num_nodes == 0 || Q.cols == 0) return {std::move(dQ), std::move(dK)};
  gf_graph_t dg = detail::device_graph(g, FusionPlan{});
  const gf_attn_desc desc = detail::step_desc<T>(kind.variant, add ? 1 : Q.cols, kind.scale,
                                                 kind.leaky_slope, !add && kind.l2_normalize_inputs);
  detail::DevBuf q = detail::DevBuf::from(Q.data), k = detail::DevBuf::from(K.data),
                 ds = detail::DevBuf::from(dS.values), gq(sizeof(T) * dQ.data.size()),
                 gk(sizeof(T) * dK.data.size());
  GFH_CALL(gf_sddmm_backward(dg, &desc, q.p, k.p, ds.p, gq.p, gk.p, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  gq.to(dQ.data);
  gk.to(dK.data);
  return {std::move(dQ), std::move(dK)};
}

template <typename T>
BackwardResult<T> unfused_backward(const Graph& g, const ForwardContext<T>& ctx,
                                   const DenseMatrix<T>& dO) {
  BackwardResult<T> r;
  r.grads = detail::backward_values(g, ctx, dO);  // the real 5-launch schedule
  r.counters = detail::backward_counter_model(g, ctx, 5);
  return r;
}

template <typename T>
BackwardResult<T> fused_backward(const Graph& g, const ForwardContext<T>& ctx,
                                 const DenseMatrix<T>& dO, const FusionPlan& plan) {
  bool feasible = true;
  if (plan.strategy == Strategy::Smmf) {
    try {
      detail::check_smmf_feasible<T>(g, plan, ctx.V.cols);
    } catch (const EngineError&) {
      feasible = false;
    }
  }
  BackwardResult<T> r;
  // feasible: the fused recompute backward (pass A + pass B); otherwise the
  // reference falls back to the unfused schedule (autograd.hpp:213-225)
  r.grads = feasible ? detail::device_backward(g, ctx, dO) : detail::backward_values(g, ctx, dO);
  r.counters = detail::backward_counters(g, ctx.V.cols, sizeof(T), feasible ? 3 : 5);
  r.counters.fallback_unfused = !feasible;
  return r;
}

template <typename T>
DenseMatrix<T> reference_forward(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                                 const DenseMatrix<T>& V, const SddmmKind& kind) {
  detail::validate_inputs(g, Q, K, V, kind);
  std::vector<T> O, lse;
  detail::device_forward(g, FusionPlan{}, Q, K, V, kind, O, lse,
                         static_cast<std::vector<T>*>(nullptr));
  DenseMatrix<T> out(g.num_nodes, V.cols);
  out.data = std::move(O);
  return out;
}

template <typename T>
T finite_difference_check(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                          const DenseMatrix<T>& V, const SddmmKind& kind, T h) {
  static_assert(sizeof(T) == 8, "finite differences require f64 inputs");
  DenseMatrix<T> Qm = Q, Km = K, Vm = V;
  auto loss = [&] {
    const auto O = reference_forward(g, Qm, Km, Vm, kind);
    T s = 0;
    for (T x : O.data) s += x;
    if (!std::isfinite(s)) throw KernelError("finite_difference_check: non-finite loss");
    return s;
  };
  ForwardContext<T> ctx;
  ctx.g = &g;
  ctx.Q = Q;
  ctx.K = K;
  ctx.V = V;
  ctx.kind = kind;
  const auto gb = detail::device_backward(g, ctx, DenseMatrix<T>(g.num_nodes, V.cols, T(1)));
  T worst = 0;
  auto probe = [&](DenseMatrix<T>& p, const DenseMatrix<T>& grad) {
    for (size_t i = 0; i < p.data.size(); ++i) {
      const T keep = p.data[i];
      p.data[i] = keep + h;
      const T up = loss();
      p.data[i] = keep - h;
      const T dn = loss();
      p.data[i] = keep;
      const T fd = (up - dn) / (2 * h);
      const T a = grad.data[i];
      worst = std::max(worst, std::abs(a - fd) / std::max({std::abs(a), std::abs(fd), T(1)}));
    }
  };
  probe(Qm, gb.dQ);
  probe(Km, gb.dK);
  probe(Vm, gb.dV);
  return worst;
}

// ----------------------------------------------------------------- models --
template <typename T>
DenseMatrix<T> matmul(const DenseMatrix<T>& A, const DenseMatrix<T>& B) {
  if (A.cols != B.rows) throw KernelError("matmul: inner dimension mismatch");
  detail::need_device();
  DenseMatrix<T> C(A.rows, B.cols);
  detail::DevBuf a = detail::DevBuf::from(A.data), b = detail::DevBuf::from(B.data);
  detail::DevBuf c(sizeof(T) * C.data.size());
  GFH_CALL(gf_gemm(detail::dtype_code<T>(), 0, A.rows, B.cols, A.cols, a.p, b.p, c.p, 0, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  c.to(C.data);
  return C;
}

template <typename T>
DenseMatrix<T> matmul_at_b(const DenseMatrix<T>& A, const DenseMatrix<T>& B) {
  if (A.rows != B.rows) throw KernelError("matmul_at_b: row count mismatch");
  detail::need_device();
  DenseMatrix<T> C(A.cols, B.cols);
  detail::DevBuf a = detail::DevBuf::from(A.data), b = detail::DevBuf::from(B.data);
  detail::DevBuf c(sizeof(T) * C.data.size());
  GFH_CALL(gf_gemm(detail::dtype_code<T>(), 1, A.cols, B.cols, A.rows, a.p, b.p, c.p, 0, nullptr));
  GFH_CALL(gf_stream_sync(nullptr));
  c.to(C.data);
  return C;
}

template <typename T>
std::pair<DenseMatrix<T>, ConvContext<T>> conv_forward(const ConvSpec& spec, const Graph& g,
                                                       const DenseMatrix<T>& X,
                                                       const ConvWeights<T>& w, FusionPlan plan) {
  const SddmmKind kind = kind_for(spec);
  plan.dtype_bytes = sizeof(T);
  plan.strategy = spec.strategy_override ? *spec.strategy_override
                                         : select_strategy(degree_stats(g), kind,
                                                           plan.shared_mem_budget_bytes,
                                                           sizeof(T));
  ConvContext<T> ctx;
  ctx.X = X;
  ForwardResult<T> res;
  if (spec.model == Model::GAT) {
    ctx.H = matmul(X, w.W_v);
    res = run_strategy(g, matmul(ctx.H, w.a_l), matmul(ctx.H, w.a_r), ctx.H, kind, plan);
  } else {
    res = run_strategy(g, matmul(X, w.W_q), matmul(X, w.W_k), matmul(X, w.W_v), kind, plan);
  }
  ctx.fwd = std::move(res.ctx);
  ctx.counters = std::move(res.counters);
  return {std::move(res.O), std::move(ctx)};
}

template <typename T>
ConvGrads<T> conv_backward(const ConvSpec& spec, const Graph& g, const ConvContext<T>& ctx,
                           const ConvWeights<T>& w, const DenseMatrix<T>& dO) {
  ConvGrads<T> out;
  out.pipeline = fused_backward(g, ctx.fwd, dO, ctx.fwd.plan).grads;
  const GradBundle<T>& gb = out.pipeline;
  if (spec.model == Model::GAT) {
    // dH = dV + del a_l^T + der a_r^T; da_l = H^T del; da_r = H^T der (models.hpp:143-150)
    detail::need_device();
    const std::int64_t n = g.num_nodes, dim = spec.dim;
    detail::DevBuf hf = detail::DevBuf::from(ctx.H.data), al = detail::DevBuf::from(w.a_l.data),
                   ar = detail::DevBuf::from(w.a_r.data), dv = detail::DevBuf::from(gb.dV.data),
                   dl = detail::DevBuf::from(gb.dQ.data), dr = detail::DevBuf::from(gb.dK.data);
    detail::DevBuf dh(sizeof(T) * n * dim), dal(sizeof(T) * dim), dar(sizeof(T) * dim);
    GFH_CALL(gf_gat_fanin(detail::dtype_code<T>(), n, 1, static_cast<std::int32_t>(dim), hf.p,
                          al.p, ar.p, dv.p, dl.p, dr.p, dh.p, dal.p, dar.p, nullptr));
    DenseMatrix<T> dW(ctx.X.cols, dim);
    detail::DevBuf x = detail::DevBuf::from(ctx.X.data), dw(sizeof(T) * dW.data.size());
    GFH_CALL(gf_gemm(detail::dtype_code<T>(), 1, ctx.X.cols, dim, n, x.p, dh.p, dw.p, 0, nullptr));
    GFH_CALL(gf_stream_sync(nullptr));
    out.da_l = DenseMatrix<T>(dim, 1);
    out.da_r = DenseMatrix<T>(dim, 1);
    dal.to(out.da_l.data);
    dar.to(out.da_r.data);
    dw.to(dW.data);
    out.dW_v = std::move(dW);
  } else {
    out.dW_q = matmul_at_b(ctx.X, gb.dQ);
    out.dW_k = matmul_at_b(ctx.X, gb.dK);
    out.dW_v = matmul_at_b(ctx.X, gb.dV);
  }
  return out;
}

template <typename T>
PipelineInputs<T> make_pipeline_inputs(const Graph& g, const ConvSpec& spec, std::uint64_t seed) {
  PipelineInputs<T> in;
  in.kind = kind_for(spec);
  in.V = random_matrix<T>(g.num_nodes, spec.dim, seed + 2);
  if (spec.model != Model::GAT) {
    in.Q = random_matrix<T>(g.num_nodes, spec.dim, seed);
    in.K = random_matrix<T>(g.num_nodes, spec.dim, seed + 1);
    return in;
  }
  // GAT: re-seed el/er until every edge pre-activation is > 1e-3 away from
  // the LeakyReLU kink (fixture rule of models.hpp:166-190).
  for (std::uint64_t bump = 0; bump < 64; ++bump) {
    in.Q = random_matrix<T>(g.num_nodes, 1, seed + bump * 1000);
    in.K = random_matrix<T>(g.num_nodes, 1, seed + 1 + bump * 1000);
    T closest = std::numeric_limits<T>::max();
    for (EdgeId k = 0; k < g.num_edges; ++k)
      closest = std::min(closest, std::abs(in.Q.data[g.coo_src[k]] + in.K.data[g.coo_dst[k]]));
    if (g.num_edges == 0 || closest > static_cast<T>(1e-3)) break;
  }
  return in;
}

#define GF_INSTANTIATE(T)                                                                        \
  template BackwardResult<T> unfused_backward<T>(const Graph&, const ForwardContext<T>&,         \
                                                 const DenseMatrix<T>&);                         \
  template BackwardResult<T> fused_backward<T>(const Graph&, const ForwardContext<T>&,           \
                                               const DenseMatrix<T>&, const FusionPlan&);        \
  template DenseMatrix<T> reference_forward<T>(const Graph&, const DenseMatrix<T>&,              \
                                               const DenseMatrix<T>&, const DenseMatrix<T>&,     \
                                               const SddmmKind&);                                \
  template DenseMatrix<T> matmul<T>(const DenseMatrix<T>&, const DenseMatrix<T>&);               \
  template DenseMatrix<T> matmul_at_b<T>(const DenseMatrix<T>&, const DenseMatrix<T>&);          \
  template std::pair<DenseMatrix<T>, ConvContext<T>> conv_forward<T>(                            \
      const ConvSpec&, const Graph&, const DenseMatrix<T>&, const ConvWeights<T>&, FusionPlan);  \
  template ConvGrads<T> conv_backward<T>(const ConvSpec&, const Graph&, const ConvContext<T>&,   \
                                         const ConvWeights<T>&, const DenseMatrix<T>&);          \
  template PipelineInputs<T> make_pipeline_inputs<T>(const Graph&, const ConvSpec&, std::uint64_t); \
  template EdgeScalars<T> sddmm_dot<T>(const Graph&, const DenseMatrix<T>&, const DenseMatrix<T>&, \
                                       T);                                                       \
  template EdgeScalars<T> sddmm_add<T>(const Graph&, const DenseMatrix<T>&, const DenseMatrix<T>&, \
                                       T);                                                       \
  template DenseMatrix<T> l2_normalize_rows<T>(const DenseMatrix<T>&, T);                        \
  template DenseMatrix<T> l2_normalize_backward<T>(const DenseMatrix<T>&, const DenseMatrix<T>&, \
                                                   T);                                           \
  template EdgeScalars<T> edge_softmax<T>(const Graph&, const EdgeScalars<T>&);                  \
  template DenseMatrix<T> spmm<T>(const Graph&, const EdgeScalars<T>&, const DenseMatrix<T>&);   \
  template EdgeScalars<T> sddmm<T>(const Graph&, const DenseMatrix<T>&, const DenseMatrix<T>&,   \
                                   const SddmmKind&);                                            \
  template std::pair<DenseMatrix<T>, DenseMatrix<T>> dense_oracle_forward<T>(                    \
      const Graph&, const DenseMatrix<T>&, const DenseMatrix<T>&, const DenseMatrix<T>&,         \
      const SddmmKind&);                                                                         \
  template std::pair<EdgeScalars<T>, DenseMatrix<T>> spmm_backward<T>(                           \
      const Graph&, const EdgeScalars<T>&, const DenseMatrix<T>&, const DenseMatrix<T>&);        \
  template EdgeScalars<T> softmax_backward<T>(const Graph&, const EdgeScalars<T>&,               \
                                              const EdgeScalars<T>&);                            \
  template std::pair<DenseMatrix<T>, DenseMatrix<T>> sddmm_backward<T>(                          \
      const Graph&, const DenseMatrix<T>&, const DenseMatrix<T>&, const EdgeScalars<T>&,         \
      const SddmmKind&);                                                                         \
  template GradBundle<T> detail::backward_values<T>(const Graph&, const ForwardContext<T>&,      \
                                                    const DenseMatrix<T>&);                      \
  template ExecCounters detail::backward_counter_model<T>(const Graph&, const ForwardContext<T>&, \
                                                          std::int64_t);

GF_INSTANTIATE(float)
GF_INSTANTIATE(double)
template double finite_difference_check<double>(const Graph&, const DenseMatrix<double>&,
                                                const DenseMatrix<double>&,
                                                const DenseMatrix<double>&, const SddmmKind&,
                                                double);

}  // namespace graphfuse

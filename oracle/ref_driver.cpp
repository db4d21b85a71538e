// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// Thin C-ABI driver over the UNMODIFIED reference implementation
// (/root/reference/proj, compiled from its own sources by oracle/Makefile into
// oracle/_ref/libgfref.so).  The reference operator API is single-head
// (SPEC.md:198); this driver loops heads over column slices so the multi-head
// B200 path can be checked against the reference's own arithmetic:
//   forward  = graphfuse::run_strategy<T>   (engine.hpp:331-336)
//   backward = graphfuse::fused_backward<T> (autograd.hpp:210-226) on a
//              context rebuilt exactly as the Python binding does
//              (module.cpp:120-130: P = edge_softmax(sddmm(Q, K))).
//   layer    = graphfuse::conv_forward / conv_backward (models.hpp:104-158)
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "graphfuse/autograd.hpp"
#include "graphfuse/engine.hpp"
#include "graphfuse/kernels.hpp"
#include "graphfuse/models.hpp"

namespace gf = graphfuse;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

gf::SddmmKind make_kind(int variant, double scale, double slope, int l2) {
  return variant == 1 ? gf::SddmmKind::add(slope) : gf::SddmmKind::dot(scale, l2 != 0);
}

// Column slice [c0, c0+w) of a row-major n x ld host buffer.
template <typename T>
gf::DenseMatrix<T> slice(const T* src, std::int64_t n, std::int64_t ld, std::int64_t c0,
                         std::int64_t w) {
  gf::DenseMatrix<T> m(n, w);
  for (std::int64_t r = 0; r < n; ++r)
    for (std::int64_t c = 0; c < w; ++c) m.data[r * w + c] = src[r * ld + c0 + c];
  return m;
}

template <typename T>
void unslice(const gf::DenseMatrix<T>& m, T* dst, std::int64_t ld, std::int64_t c0) {
  for (std::int64_t r = 0; r < m.rows; ++r)
    for (std::int64_t c = 0; c < m.cols; ++c) dst[r * ld + c0 + c] = m.data[r * m.cols + c];
}

// Per-head operand widths: dot -> Q,K are N x (H*D); add -> el,er are N x H.
struct Shape {
  std::int64_t n, H, D, qk_ld, qk_w;
};

Shape shape_of(const gf::Graph& g, int H, int D, int variant) {
  Shape s{g.num_nodes, H, D, variant == 1 ? H : std::int64_t(H) * D, variant == 1 ? 1 : D};
  return s;
}

template <typename T>
int forward_impl(const gf::Graph* g, int H, int D, int variant, double scale, double slope,
                 int l2, int strategy, std::int64_t budget, const T* Q, const T* K, const T* V,
                 T* O, T* P, std::uint64_t* elapsed_ns) {
  try {
    Shape sh = shape_of(*g, H, D, variant);
    gf::FusionPlan plan;
    plan.dtype_bytes = sizeof(T);
    plan.strategy = static_cast<gf::Strategy>(strategy);
    plan.shared_mem_budget_bytes = budget;
    auto kind = make_kind(variant, scale, slope, l2);
    std::uint64_t total = 0;
    for (int h = 0; h < H; ++h) {
      auto q = slice(Q, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      auto k = slice(K, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      auto v = slice(V, sh.n, std::int64_t(H) * D, std::int64_t(h) * D, D);
      auto res = gf::run_strategy(*g, q, k, v, kind, plan);
      total += res.counters.elapsed_ns;
      unslice(res.O, O, std::int64_t(H) * D, std::int64_t(h) * D);
      if (P)
        for (gf::EdgeId e = 0; e < g->num_edges; ++e) P[e * H + h] = res.ctx.P[e];
    }
    if (elapsed_ns) *elapsed_ns = total;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

template <typename T>
int backward_impl(const gf::Graph* g, int H, int D, int variant, double scale, double slope,
                  int l2, int fused, const T* Q, const T* K, const T* V, const T* dO, T* dQ,
                  T* dK, T* dV, std::uint64_t* counters5) {
  try {
    Shape sh = shape_of(*g, H, D, variant);
    auto kind = make_kind(variant, scale, slope, l2);
    for (int h = 0; h < H; ++h) {
      gf::ForwardContext<T> ctx;
      ctx.g = g;
      ctx.Q = slice(Q, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      ctx.K = slice(K, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      ctx.V = slice(V, sh.n, std::int64_t(H) * D, std::int64_t(h) * D, D);
      ctx.kind = kind;
      ctx.P = gf::edge_softmax(*g, gf::sddmm(*g, ctx.Q, ctx.K, kind));
      auto d_o = slice(dO, sh.n, std::int64_t(H) * D, std::int64_t(h) * D, D);
      auto res = fused ? gf::fused_backward(*g, ctx, d_o, gf::FusionPlan{})
                       : gf::unfused_backward(*g, ctx, d_o);
      unslice(res.grads.dQ, dQ, sh.qk_ld, h * sh.qk_w);
      unslice(res.grads.dK, dK, sh.qk_ld, h * sh.qk_w);
      unslice(res.grads.dV, dV, std::int64_t(H) * D, std::int64_t(h) * D);
      if (counters5 && h == 0) {
        counters5[0] = res.counters.kernel_launches;
        counters5[1] = res.counters.global_bytes_read;
        counters5[2] = res.counters.global_bytes_written;
        counters5[3] = res.counters.fallback_unfused ? 1 : 0;
        counters5[4] = 0;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Timing leg for the CPU baseline: the reference forward (run_strategy) and
// backward (fused_backward on the saved forward context) for ONE head, each
// timed with steady_clock around the reference call only.
template <typename T>
int time_head_impl(const gf::Graph* g, int D, int variant, double scale, double slope, int l2,
                   const T* Q, const T* K, const T* V, const T* dO, double* fwd_s,
                   double* bwd_s) {
  try {
    std::int64_t w = variant == 1 ? 1 : D;
    gf::DenseMatrix<T> q(g->num_nodes, w), k(g->num_nodes, w), v(g->num_nodes, D),
        d_o(g->num_nodes, D);
    std::memcpy(q.data.data(), Q, sizeof(T) * q.data.size());
    std::memcpy(k.data.data(), K, sizeof(T) * k.data.size());
    std::memcpy(v.data.data(), V, sizeof(T) * v.data.size());
    std::memcpy(d_o.data.data(), dO, sizeof(T) * d_o.data.size());
    gf::FusionPlan plan;
    plan.dtype_bytes = sizeof(T);
    plan.shared_mem_budget_bytes = std::int64_t(1) << 30;  // numerics-only precedent, acceptance_main.cpp:46
    auto kind = make_kind(variant, scale, slope, l2);
    auto t0 = std::chrono::steady_clock::now();
    auto res = gf::run_strategy(*g, q, k, v, kind, plan);
    auto t1 = std::chrono::steady_clock::now();
    auto bw = gf::fused_backward(*g, res.ctx, d_o, plan);
    auto t2 = std::chrono::steady_clock::now();
    *fwd_s = std::chrono::duration<double>(t1 - t0).count();
    *bwd_s = std::chrono::duration<double>(t2 - t1).count();
    volatile T sink = res.O.data.empty() ? T(0) : res.O.data[0];
    sink = bw.grads.dV.data.empty() ? T(0) : bw.grads.dV.data[0];
    (void)sink;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Timing leg of the reference arm: one whole multi-head layer step, every
// head h = 0..H-1 through run_strategy<T> then fused_backward<T> (the
// reference is single-head, so a multi-head user slices columns
// per head).  Only the reference calls are timed; the column slicing is not.
template <typename T>
int time_step_impl(const gf::Graph* g, int H, int D, int variant, double scale, double slope,
                   int l2, const T* Q, const T* K, const T* V, const T* dO, double* fwd_s,
                   double* bwd_s) {
  try {
    Shape sh = shape_of(*g, H, D, variant);
    gf::FusionPlan plan;
    plan.dtype_bytes = sizeof(T);
    plan.shared_mem_budget_bytes = std::int64_t(1) << 30;  // acceptance_main.cpp:46 precedent
    auto kind = make_kind(variant, scale, slope, l2);
    double f = 0, b = 0;
    volatile T sink = 0;
    for (int h = 0; h < H; ++h) {
      auto q = slice(Q, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      auto k = slice(K, sh.n, sh.qk_ld, h * sh.qk_w, sh.qk_w);
      auto v = slice(V, sh.n, std::int64_t(H) * D, std::int64_t(h) * D, D);
      auto d_o = slice(dO, sh.n, std::int64_t(H) * D, std::int64_t(h) * D, D);
      auto t0 = std::chrono::steady_clock::now();
      auto res = gf::run_strategy(*g, q, k, v, kind, plan);
      auto t1 = std::chrono::steady_clock::now();
      auto bw = gf::fused_backward(*g, res.ctx, d_o, plan);
      auto t2 = std::chrono::steady_clock::now();
      f += std::chrono::duration<double>(t1 - t0).count();
      b += std::chrono::duration<double>(t2 - t1).count();
      sink = res.O.data.empty() ? T(0) : res.O.data[0];
      sink = bw.grads.dV.data.empty() ? T(0) : bw.grads.dV.data[0];
    }
    (void)sink;
    *fwd_s = f;
    *bwd_s = b;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Layer level (models.hpp:104-158), every head: conv_forward + conv_backward
// with head h's weight columns (W[:, hD:(h+1)D], a_l/a_r[hD:(h+1)D]).  X is
// N x d_in; dO is N x (H*D).  *pipe_s = the part of that time spent in
// run_strategy + fused_backward (timed separately on the same inputs), so a
// caller can split projection and pipeline cost.
template <typename T>
int time_conv_impl(const gf::Graph* g, int model, int H, std::int64_t D, std::int64_t d_in,
                   double scale, double slope, const T* X, const T* Wq, const T* Wk, const T* Wv,
                   const T* al, const T* ar, const T* dO, double* layer_s) {
  try {
    gf::ConvSpec spec;
    spec.model = static_cast<gf::Model>(model);
    spec.dim = D;
    spec.scale = scale;
    spec.leaky_slope = slope;
    gf::DenseMatrix<T> x(g->num_nodes, d_in);
    std::memcpy(x.data.data(), X, sizeof(T) * x.data.size());
    gf::FusionPlan plan;
    plan.dtype_bytes = sizeof(T);
    plan.shared_mem_budget_bytes = std::int64_t(1) << 30;
    const std::int64_t F = std::int64_t(H) * D;
    double t = 0;
    volatile T sink = 0;
    for (int h = 0; h < H; ++h) {
      gf::ConvWeights<T> w;
      w.W_v = slice(Wv, d_in, F, h * D, D);
      if (spec.model == gf::Model::GAT) {
        gf::DenseMatrix<T> a(D, 1), b(D, 1);
        for (std::int64_t i = 0; i < D; ++i) {
          a.data[i] = al[h * D + i];
          b.data[i] = ar[h * D + i];
        }
        w.a_l = a;
        w.a_r = b;
      } else {
        w.W_q = slice(Wq, d_in, F, h * D, D);
        w.W_k = slice(Wk, d_in, F, h * D, D);
      }
      auto d_o = slice(dO, g->num_nodes, F, h * D, D);
      auto t0 = std::chrono::steady_clock::now();
      auto [out, ctx] = gf::conv_forward(spec, *g, x, w, plan);
      auto grads = gf::conv_backward(spec, *g, ctx, w, d_o);
      auto t1 = std::chrono::steady_clock::now();
      t += std::chrono::duration<double>(t1 - t0).count();
      sink = out.data.empty() ? T(0) : out.data[0];
      sink = grads.dW_v.data.empty() ? T(0) : grads.dW_v.data[0];
    }
    (void)sink;
    *layer_s = t;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // namespace

extern "C" {

const char* gfref_last_error() { return g_err.c_str(); }

void* gfref_from_coo(std::int64_t n, std::int64_t e, const std::int64_t* src,
                     const std::int64_t* dst) {
  try {
    std::vector<gf::NodeId> s(src, src + e), d(dst, dst + e);
    return new gf::Graph(gf::from_coo(n, s, d));
  } catch (const std::exception& ex) {
    fail(ex);
    return nullptr;
  }
}

// Adopt an already-canonical CSR/CSC (used by the CPU baseline at Reddit scale
// so the timed reference run does not pay the 17 s single-threaded from_coo).
void* gfref_graph_adopt(std::int64_t n, std::int64_t e, const std::int64_t* row_ptr,
                        const std::int64_t* col, const std::int64_t* csc_ptr,
                        const std::int64_t* csc_row, const std::int64_t* csc_perm) {
  auto* g = new gf::Graph();
  g->num_nodes = n;
  g->num_edges = e;
  g->csr_row_ptr.assign(row_ptr, row_ptr + n + 1);
  g->csr_col_idx.assign(col, col + e);
  g->coo_src = g->csr_col_idx;
  g->coo_dst.resize(e);
  for (std::int64_t v = 0; v < n; ++v)
    for (std::int64_t i = row_ptr[v]; i < row_ptr[v + 1]; ++i) g->coo_dst[i] = v;
  g->csc_col_ptr.assign(csc_ptr, csc_ptr + n + 1);
  g->csc_row_idx.assign(csc_row, csc_row + e);
  g->csc_edge_perm.assign(csc_perm, csc_perm + e);
  return g;
}

void* gfref_gen_random(std::int64_t n, double avg, std::uint64_t seed) {
  try {
    return new gf::Graph(gf::gen_random(n, avg, seed));
  } catch (const std::exception& ex) {
    fail(ex);
    return nullptr;
  }
}

void* gfref_gen_super_node(std::int64_t n, double avg, std::int64_t hub, std::uint64_t seed) {
  try {
    return new gf::Graph(gf::gen_super_node(n, avg, hub, seed));
  } catch (const std::exception& ex) {
    fail(ex);
    return nullptr;
  }
}

void gfref_graph_free(void* g) { delete static_cast<gf::Graph*>(g); }
std::int64_t gfref_num_nodes(void* g) { return static_cast<gf::Graph*>(g)->num_nodes; }
std::int64_t gfref_num_edges(void* g) { return static_cast<gf::Graph*>(g)->num_edges; }

void gfref_graph_arrays(void* gp, std::int64_t* row_ptr, std::int64_t* col,
                        std::int64_t* csc_ptr, std::int64_t* csc_row, std::int64_t* csc_perm) {
  auto* g = static_cast<gf::Graph*>(gp);
  auto cp = [](const std::vector<std::int64_t>& v, std::int64_t* out) {
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
  };
  cp(g->csr_row_ptr, row_ptr);
  cp(g->csr_col_idx, col);
  cp(g->csc_col_ptr, csc_ptr);
  cp(g->csc_row_idx, csc_row);
  cp(g->csc_edge_perm, csc_perm);
}

int gfref_forward_f32(void* g, int H, int D, int variant, double scale, double slope, int l2,
                      int strategy, std::int64_t budget, const float* Q, const float* K,
                      const float* V, float* O, float* P, std::uint64_t* elapsed_ns) {
  return forward_impl<float>(static_cast<gf::Graph*>(g), H, D, variant, scale, slope, l2,
                             strategy, budget, Q, K, V, O, P, elapsed_ns);
}
int gfref_forward_f64(void* g, int H, int D, int variant, double scale, double slope, int l2,
                      int strategy, std::int64_t budget, const double* Q, const double* K,
                      const double* V, double* O, double* P, std::uint64_t* elapsed_ns) {
  return forward_impl<double>(static_cast<gf::Graph*>(g), H, D, variant, scale, slope, l2,
                              strategy, budget, Q, K, V, O, P, elapsed_ns);
}
int gfref_backward_f32(void* g, int H, int D, int variant, double scale, double slope, int l2,
                       int fused, const float* Q, const float* K, const float* V,
                       const float* dO, float* dQ, float* dK, float* dV, std::uint64_t* c5) {
  return backward_impl<float>(static_cast<gf::Graph*>(g), H, D, variant, scale, slope, l2,
                              fused, Q, K, V, dO, dQ, dK, dV, c5);
}
int gfref_backward_f64(void* g, int H, int D, int variant, double scale, double slope, int l2,
                       int fused, const double* Q, const double* K, const double* V,
                       const double* dO, double* dQ, double* dK, double* dV,
                       std::uint64_t* c5) {
  return backward_impl<double>(static_cast<gf::Graph*>(g), H, D, variant, scale, slope, l2,
                               fused, Q, K, V, dO, dQ, dK, dV, c5);
}
int gfref_time_head_f32(void* g, int D, int variant, double scale, double slope, int l2,
                        const float* Q, const float* K, const float* V, const float* dO,
                        double* fwd_s, double* bwd_s) {
  return time_head_impl<float>(static_cast<gf::Graph*>(g), D, variant, scale, slope, l2, Q, K,
                               V, dO, fwd_s, bwd_s);
}

int gfref_time_step_f32(void* g, int H, int D, int variant, double scale, double slope, int l2,
                        const float* Q, const float* K, const float* V, const float* dO,
                        double* fwd_s, double* bwd_s) {
  return time_step_impl<float>(static_cast<gf::Graph*>(g), H, D, variant, scale, slope, l2, Q,
                               K, V, dO, fwd_s, bwd_s);
}
int gfref_time_conv_f32(void* g, int model, int H, std::int64_t D, std::int64_t d_in,
                        double scale, double slope, const float* X, const float* Wq,
                        const float* Wk, const float* Wv, const float* al, const float* ar,
                        const float* dO, double* layer_s) {
  return time_conv_impl<float>(static_cast<gf::Graph*>(g), model, H, D, d_in, scale, slope, X,
                               Wq, Wk, Wv, al, ar, dO, layer_s);
}

// Counters of one single-head forward (ExecCounters::to_map order, elapsed excluded):
// gbr, gbw, shared, tx, launches, softmax_ops, s, f, p, max_group_load, fallback.
// per_group loads copied to loads (capacity cap), count returned in *n_loads.
int gfref_forward_counters(void* gp, int d, int variant, int l2, int strategy,
                           std::int64_t rows_per_block, std::int64_t groups,
                           std::int64_t group_width, std::int64_t vector_width,
                           std::int64_t budget, int dtype_bytes, std::uint64_t* out11,
                           std::uint64_t* loads, std::int64_t cap, std::int64_t* n_loads) {
  try {
    auto* g = static_cast<gf::Graph*>(gp);
    gf::FusionPlan plan;
    plan.strategy = static_cast<gf::Strategy>(strategy);
    plan.rows_per_block = rows_per_block;
    plan.groups_per_block = groups;
    plan.group_width = group_width;
    plan.vector_width = vector_width;
    plan.shared_mem_budget_bytes = budget;
    plan.dtype_bytes = dtype_bytes;
    auto kind = make_kind(variant, 1.0, 0.2, l2);
    std::int64_t w = variant == 1 ? 1 : d;
    gf::ExecCounters c;
    if (dtype_bytes == 8) {
      auto q = gf::random_matrix<double>(g->num_nodes, w, 1);
      auto v = gf::random_matrix<double>(g->num_nodes, d, 3);
      c = gf::run_strategy(*g, q, q, v, kind, plan).counters;
    } else {
      auto q = gf::random_matrix<float>(g->num_nodes, w, 1);
      auto v = gf::random_matrix<float>(g->num_nodes, d, 3);
      c = gf::run_strategy(*g, q, q, v, kind, plan).counters;
    }
    auto m = c.to_map(false);
    const char* keys[11] = {"global_bytes_read", "global_bytes_written", "shared_bytes_accessed",
                            "memory_transactions", "kernel_launches", "softmax_scalar_ops",
                            "s_global_bytes", "f_global_bytes", "p_global_bytes",
                            "max_group_load", "fallback_unfused"};
    for (int i = 0; i < 11; ++i) out11[i] = m[keys[i]];
    *n_loads = static_cast<std::int64_t>(c.per_group_edge_loads.size());
    for (std::int64_t i = 0; i < cap && i < *n_loads; ++i) loads[i] = c.per_group_edge_loads[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Layer level, single head (models.hpp:104-158). model: 0 GT, 1 AGNN, 2 GAT.
// Weights: Wq, Wk, Wv are d_in x dim; a_l, a_r are dim (GAT).  dO is N x dim.
int gfref_conv_f64(void* gp, int model, std::int64_t dim, std::int64_t d_in, double scale,
                   double slope, const double* X, const double* Wq, const double* Wk,
                   const double* Wv, const double* al, const double* ar, const double* dO,
                   double* O, double* dWq, double* dWk, double* dWv, double* dal, double* dar) {
  try {
    auto* g = static_cast<gf::Graph*>(gp);
    gf::ConvSpec spec;
    spec.model = static_cast<gf::Model>(model);
    spec.dim = dim;
    spec.scale = scale;
    spec.leaky_slope = slope;
    auto mat = [](const double* p, std::int64_t r, std::int64_t c) {
      gf::DenseMatrix<double> m(r, c);
      if (p) std::memcpy(m.data.data(), p, sizeof(double) * r * c);
      return m;
    };
    gf::DenseMatrix<double> x = mat(X, g->num_nodes, d_in);
    gf::ConvWeights<double> w;
    w.W_v = mat(Wv, d_in, dim);
    if (spec.model == gf::Model::GAT) {
      w.a_l = mat(al, dim, 1);
      w.a_r = mat(ar, dim, 1);
    } else {
      w.W_q = mat(Wq, d_in, dim);
      w.W_k = mat(Wk, d_in, dim);
    }
    gf::FusionPlan plan;
    plan.shared_mem_budget_bytes = std::int64_t(1) << 30;
    auto [out, ctx] = gf::conv_forward(spec, *g, x, w, plan);
    std::memcpy(O, out.data.data(), sizeof(double) * out.data.size());
    auto grads = gf::conv_backward(spec, *g, ctx, w, mat(dO, g->num_nodes, dim));
    auto put = [](const gf::DenseMatrix<double>& m, double* p) {
      if (p && !m.data.empty()) std::memcpy(p, m.data.data(), sizeof(double) * m.data.size());
    };
    put(grads.dW_v, dWv);
    put(grads.dW_q, dWq);
    put(grads.dW_k, dWk);
    put(grads.da_l, dal);
    put(grads.da_r, dar);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double gfref_gradcheck(void* gp, int model, std::int64_t dim, std::uint64_t seed, double h) {
  auto* g = static_cast<gf::Graph*>(gp);
  gf::ConvSpec spec;
  spec.model = static_cast<gf::Model>(model);
  spec.dim = dim;
  auto in = gf::make_pipeline_inputs<double>(*g, spec, seed);
  return gf::finite_difference_check(*g, in.Q, in.K, in.V, in.kind, h);
}

// random_matrix (dense.hpp:78-86) so tests can reproduce reference fixtures.
void gfref_random_matrix_f64(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double lo,
                             double hi, double* out) {
  auto m = gf::random_matrix<double>(rows, cols, seed, lo, hi);
  std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
}
void gfref_random_matrix_f32(std::int64_t rows, std::int64_t cols, std::uint64_t seed, float lo,
                             float hi, float* out) {
  auto m = gf::random_matrix<float>(rows, cols, seed, lo, hi);
  std::memcpy(out, m.data.data(), sizeof(float) * m.data.size());
}

}  // extern "C"

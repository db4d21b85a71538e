// Timing of the reference-facing C++ operator API itself ("time
// the drop-in API path once"): what a reference user pays for one multi-head
// layer step through the unchanged single-head templates, i.e. for every head
// run_strategy<T> (engine.hpp:331-336: host Q/K/V uploaded, forward, O and P
// downloaded, counters modelled) then fused_backward<T> (autograd.hpp:210-226:
// context uploaded, recompute backward, gradients downloaded).  Exposed as a
// plain C symbol for bench.py (ctypes); not part of the reference API.
#include <chrono>
#include <cstring>
#include <random>

#include "graphfuse/graphfuse.hpp"

namespace {

template <typename T>
graphfuse::DenseMatrix<T> random_cols(std::int64_t n, std::int64_t w, std::uint64_t seed) {
  graphfuse::DenseMatrix<T> m(n, w);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  for (T& x : m.data) x = static_cast<T>(d(rng));
  return m;
}

}  // namespace

extern "C" int gfh_time_api_step(std::int64_t n, std::int64_t e, const std::int64_t* row_ptr,
                                 const std::int64_t* col, const std::int64_t* csc_ptr,
                                 const std::int64_t* csc_row, const std::int64_t* csc_perm,
                                 int heads, int head_dim, int variant, int reps, double* fwd_ms,
                                 double* bwd_ms, char* err, int err_len) {
  namespace gf = graphfuse;
  try {
    gf::Graph g;
    g.num_nodes = n;
    g.num_edges = e;
    g.csr_row_ptr.assign(row_ptr, row_ptr + n + 1);
    g.csr_col_idx.assign(col, col + e);
    g.coo_src = g.csr_col_idx;
    g.coo_dst.resize(static_cast<size_t>(e));
    for (std::int64_t v = 0; v < n; ++v)
      for (std::int64_t i = row_ptr[v]; i < row_ptr[v + 1]; ++i) g.coo_dst[i] = v;
    g.csc_col_ptr.assign(csc_ptr, csc_ptr + n + 1);
    g.csc_row_idx.assign(csc_row, csc_row + e);
    g.csc_edge_perm.assign(csc_perm, csc_perm + e);
    const gf::SddmmKind kind = variant == 1 ? gf::SddmmKind::add(0.2)
                                            : gf::SddmmKind::dot(1.0 / std::sqrt(double(head_dim)));
    const std::int64_t qk = variant == 1 ? 1 : head_dim;
    gf::FusionPlan plan;
    plan.shared_mem_budget_bytes = std::int64_t(1) << 30;  // acceptance_main.cpp:46 precedent
    std::vector<gf::DenseMatrix<float>> Q, K, V, dO;
    for (int h = 0; h < heads; ++h) {
      Q.push_back(random_cols<float>(n, qk, 10 + h));
      K.push_back(random_cols<float>(n, qk, 20 + h));
      V.push_back(random_cols<float>(n, head_dim, 30 + h));
      dO.push_back(random_cols<float>(n, head_dim, 40 + h));
    }
    double f = 0, b = 0;
    for (int r = -1; r < reps; ++r) {  // r = -1: warm-up (device graph upload, pools)
      for (int h = 0; h < heads; ++h) {
        auto t0 = std::chrono::steady_clock::now();
        auto fr = gf::run_strategy(g, Q[h], K[h], V[h], kind, plan);
        auto t1 = std::chrono::steady_clock::now();
        auto br = gf::fused_backward(g, fr.ctx, dO[h], plan);
        auto t2 = std::chrono::steady_clock::now();
        if (r >= 0) {
          f += std::chrono::duration<double, std::milli>(t1 - t0).count();
          b += std::chrono::duration<double, std::milli>(t2 - t1).count();
        }
      }
    }
    *fwd_ms = f / std::max(1, reps);
    *bwd_ms = b / std::max(1, reps);
    return 0;
  } catch (const std::exception& ex) {
    if (err && err_len > 0) {
      std::strncpy(err, ex.what(), static_cast<size_t>(err_len - 1));
      err[err_len - 1] = 0;
    }
    return 1;
  }
}

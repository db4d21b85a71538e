// graphfuse.hpp — B200-native drop-in for the reference's C++ operator API.
//
// Same namespace, type names, function names, argument meaning and error
// behaviour as the reference `graphfuse` headers (/root/reference/proj/
// include/graphfuse/*.hpp); the compute underneath is the sm_100a path in
// libgraphfuse_cuda.so, reached ONLY through the C-ABI in gf_cuda.h.  There
// is no CPU compute fallback: if the CUDA library or device is unavailable
// every compute entry point throws EngineError.
//
// Drop-in map (reference file:line -> here):
//   graph.hpp:24-75      Graph, DegreeStats, from_coo, degree_stats, ...
//   dense.hpp:18-86      DenseMatrix, EdgeScalars, SddmmKind, random_matrix
//   schedule.hpp:12-75   Strategy, FusionPlan, planners
//   counters.hpp:17-67   ExecCounters (modelled counters kept byte-identical)
//   engine.hpp:25-336    ForwardContext/Result, run_smmf/pmf/.../run_strategy
//   autograd.hpp:19-287  GradBundle, BackwardResult, fused/unfused_backward,
//                        finite_difference_check
//   models.hpp:17-197    Model, ConvSpec, ConvWeights/Context/Grads,
//                        conv_forward/backward, make_pipeline_inputs, ...
// The old per-file include paths are kept as one-line forwarding headers.
#pragma once

#include <cmath>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace graphfuse {

using NodeId = std::int64_t;
using EdgeId = std::int64_t;

struct GraphError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct KernelError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct EngineError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
struct DeviceGraphCache;  // device CSR/CSC + schedules, built on first use
}

// ------------------------------------------------------------------ graph --
/// Hybrid CSR (destination rows, sources sorted) + COO (CSR order) + CSC
/// (source columns, destinations sorted; csc_edge_perm = CSR edge id).
struct Graph {
  NodeId num_nodes = 0;
  EdgeId num_edges = 0;
  std::vector<EdgeId> csr_row_ptr;
  std::vector<NodeId> csr_col_idx;
  std::vector<NodeId> coo_dst;
  std::vector<NodeId> coo_src;
  std::vector<EdgeId> csc_col_ptr;
  std::vector<NodeId> csc_row_idx;
  std::vector<EdgeId> csc_edge_perm;

  NodeId in_degree(NodeId v) const { return csr_row_ptr[v + 1] - csr_row_ptr[v]; }
  NodeId out_degree(NodeId u) const { return csc_col_ptr[u + 1] - csc_col_ptr[u]; }

  /// B200: device-resident copy of the topology, uploaded once per Graph.
  mutable std::shared_ptr<detail::DeviceGraphCache> device;
};

struct DegreeStats {
  double avg_degree = 0.0;
  NodeId max_degree = 0;
  NodeId min_degree = 0;
};

Graph from_coo(NodeId num_nodes, const std::vector<NodeId>& src, const std::vector<NodeId>& dst);
DegreeStats degree_stats(const Graph& g);
std::int64_t super_node_threshold(std::int64_t shared_mem_bytes, std::int64_t dtype_bytes);
bool has_super_node(const DegreeStats& stats, std::int64_t shared_mem_bytes,
                    std::int64_t dtype_bytes);
Graph batch_graphs(const std::vector<Graph>& gs);
Graph gen_random(NodeId n, double avg_degree, std::uint64_t seed);
Graph gen_super_node(NodeId n, double avg_degree, NodeId hub_degree, std::uint64_t seed);
void write_graph(std::ostream& os, const Graph& g);
Graph read_graph(std::istream& is);
void save_graph(const std::string& path, const Graph& g);
Graph load_graph(const std::string& path);

// ------------------------------------------------------------------ dense --
template <typename T>
struct DenseMatrix {
  std::int64_t rows = 0;
  std::int64_t cols = 0;
  std::vector<T> data;
  DenseMatrix() = default;
  DenseMatrix(std::int64_t r, std::int64_t c, T fill = T(0))
      : rows(r), cols(c), data(static_cast<size_t>(r * c), fill) {}
  T* row(std::int64_t r) { return data.data() + r * cols; }
  const T* row(std::int64_t r) const { return data.data() + r * cols; }
  T& at(std::int64_t r, std::int64_t c) { return data[r * cols + c]; }
  T at(std::int64_t r, std::int64_t c) const { return data[r * cols + c]; }
};

template <typename T>
struct EdgeScalars {
  std::vector<T> values;
  EdgeScalars() = default;
  explicit EdgeScalars(EdgeId e, T fill = T(0)) : values(static_cast<size_t>(e), fill) {}
  EdgeId size() const { return static_cast<EdgeId>(values.size()); }
  T& operator[](EdgeId e) { return values[static_cast<size_t>(e)]; }
  T operator[](EdgeId e) const { return values[static_cast<size_t>(e)]; }
};

enum class SddmmVariant { Dot, Add };

struct SddmmKind {
  SddmmVariant variant = SddmmVariant::Dot;
  double scale = 1.0;
  double leaky_slope = 0.2;
  bool l2_normalize_inputs = false;
  static SddmmKind dot(double scale = 1.0, bool l2 = false) {
    return {SddmmVariant::Dot, scale, 0.2, l2};
  }
  static SddmmKind add(double slope = 0.2) { return {SddmmVariant::Add, 1.0, slope, false}; }
};

template <typename T>
bool all_finite(const DenseMatrix<T>& m) {
  for (T v : m.data)
    if (!std::isfinite(v)) return false;
  return true;
}

template <typename T>
bool all_finite(const EdgeScalars<T>& s) {
  for (T v : s.values)
    if (!std::isfinite(v)) return false;
  return true;
}

/// Uniform [lo, hi) fixture matrix from mt19937_64 (same stream as dense.hpp:78-86).
template <typename T>
DenseMatrix<T> random_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed,
                             T lo = T(-1), T hi = T(1)) {
  DenseMatrix<T> m(rows, cols);
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(lo, hi);
  for (auto& x : m.data) x = static_cast<T>(u(gen));
  return m;
}

// --------------------------------------------------------------- schedule --
enum class Strategy { Smmf, Pmf, Unfused, FeatureParallelBaseline };
std::string to_string(Strategy s);
Strategy strategy_from_string(const std::string& name);

struct FusionPlan {
  Strategy strategy = Strategy::Smmf;
  std::int64_t rows_per_block = 4;
  std::int64_t groups_per_block = 4;
  std::int64_t group_width = 32;
  std::int64_t vector_width = 4;
  std::int64_t shared_mem_budget_bytes = 49152;
  std::int64_t dtype_bytes = 4;
  bool deterministic = false;
  /// B200: rows with in-degree >= this run as an 8-warp edge-split CTA
  /// (0 = library default).  Does not change results beyond rounding order.
  std::int64_t cta_row_threshold = 0;
  FusionPlan with_strategy(Strategy s) const {
    FusionPlan p = *this;
    p.strategy = s;
    return p;
  }
};

struct RowRange {
  NodeId begin = 0;
  NodeId end = 0;
};
struct EdgeRange {
  EdgeId begin = 0;
  EdgeId end = 0;
  EdgeId size() const { return end - begin; }
};
struct BlockAssignment {
  std::int64_t block_id = 0;
  RowRange rows;
  std::vector<EdgeRange> per_group_edges;
};

Strategy select_strategy(const DegreeStats& stats, const SddmmKind& kind,
                         std::int64_t shared_mem_bytes, std::int64_t dtype_bytes);
std::vector<RowRange> partition_blocks(const Graph& g, std::int64_t rows_per_block);
BlockAssignment warp_balance(const Graph& g, const RowRange& rows, std::int64_t groups_per_block);
std::vector<EdgeRange> edge_parallel_partition(const Graph& g, std::int64_t num_blocks);
std::int64_t shared_mem_usage(const FusionPlan& plan, std::int64_t block_max_edges,
                              std::int64_t d);
std::int64_t pmf_sddmm_block_count(const Graph& g, const FusionPlan& plan);

// --------------------------------------------------------------- counters --
/// Modelled execution counters (the reference's analytic model, unchanged so
/// drop-in tests keep passing) plus the B200 measurement of the device time.
struct ExecCounters {
  std::uint64_t global_bytes_read = 0;
  std::uint64_t global_bytes_written = 0;
  std::uint64_t shared_bytes_accessed = 0;
  std::uint64_t memory_transactions = 0;
  std::uint64_t kernel_launches = 0;
  std::uint64_t softmax_scalar_ops = 0;
  std::uint64_t s_global_bytes = 0;
  std::uint64_t f_global_bytes = 0;
  std::uint64_t p_global_bytes = 0;
  std::vector<std::uint64_t> per_group_edge_loads;
  std::uint64_t elapsed_ns = 0;
  bool fallback_unfused = false;

  std::uint64_t max_group_load() const;
  double mean_group_load() const;
  std::map<std::string, std::uint64_t> to_map(bool include_elapsed = true) const;
  bool same_model(const ExecCounters& o) const;
};

inline std::int64_t vectorized_transactions(std::int64_t d, std::int64_t vector_width) {
  return (d + vector_width - 1) / vector_width;
}

// ----------------------------------------------------------------- engine --
template <typename T>
struct ForwardContext {
  const Graph* g = nullptr;
  DenseMatrix<T> Q, K, V;
  EdgeScalars<T> P;
  SddmmKind kind;
  FusionPlan plan;
  /// B200: forward statistics for the recompute backward (O and the
  /// per-row softmax statistics (max, log-sum), 2 per row).  Empty when the
  /// context is built by hand; the
  /// backward then recomputes them on the device.
  std::vector<T> O, lse;
};

template <typename T>
struct ForwardResult {
  DenseMatrix<T> O;
  ForwardContext<T> ctx;
  ExecCounters counters;
};

namespace detail {
template <typename T>
ExecCounters model_counters(const Graph& g, const SddmmKind& kind, const FusionPlan& plan,
                            std::int64_t d, Strategy mode);
template <typename T>
void check_smmf_feasible(const Graph& g, const FusionPlan& plan, std::int64_t d);
template <typename T>
ForwardResult<T> run_mode(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                          const DenseMatrix<T>& V, const SddmmKind& kind, const FusionPlan& plan,
                          Strategy mode);
}  // namespace detail

template <typename T>
ForwardResult<T> run_smmf(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                          const DenseMatrix<T>& V, const SddmmKind& kind, const FusionPlan& plan) {
  return detail::run_mode(g, Q, K, V, kind, plan, Strategy::Smmf);
}
template <typename T>
ForwardResult<T> run_pmf(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                         const DenseMatrix<T>& V, const SddmmKind& kind, const FusionPlan& plan) {
  return detail::run_mode(g, Q, K, V, kind, plan, Strategy::Pmf);
}
template <typename T>
ForwardResult<T> run_feature_parallel_baseline(const Graph& g, const DenseMatrix<T>& Q,
                                               const DenseMatrix<T>& K, const DenseMatrix<T>& V,
                                               const SddmmKind& kind, const FusionPlan& plan) {
  return detail::run_mode(g, Q, K, V, kind, plan, Strategy::FeatureParallelBaseline);
}
template <typename T>
ForwardResult<T> run_unfused(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                             const DenseMatrix<T>& V, const SddmmKind& kind,
                             const FusionPlan& plan = FusionPlan{}) {
  return detail::run_mode(g, Q, K, V, kind, plan, Strategy::Unfused);
}
template <typename T>
ForwardResult<T> run_strategy(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                              const DenseMatrix<T>& V, const SddmmKind& kind,
                              const FusionPlan& plan) {
  return detail::run_mode(g, Q, K, V, kind, plan, plan.strategy);
}

// ----------------------------------------------------------- kernels.hpp --
// Single-step operators (kernels.hpp:18-117), each one device op
// (gf_sddmm / gf_edge_softmax / gf_spmm / gf_l2_normalize_rows), and the
// reference's masked dense oracle dense_oracle_forward (kernels.hpp:122-166)
// as a dense device op (gf_dense_oracle_forward; N <= 4096, KernelError
// "dense_oracle_forward: N > 4096" otherwise).  Returns (S_dense, O) with
// S_dense[v][u] the score of edge u -> v.
template <typename T>
EdgeScalars<T> sddmm_dot(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                         T scale);
template <typename T>
EdgeScalars<T> sddmm_add(const Graph& g, const DenseMatrix<T>& el, const DenseMatrix<T>& er,
                         T leaky_slope);
template <typename T>
DenseMatrix<T> l2_normalize_rows(const DenseMatrix<T>& X, T eps);
template <typename T>
EdgeScalars<T> edge_softmax(const Graph& g, const EdgeScalars<T>& s);
template <typename T>
DenseMatrix<T> spmm(const Graph& g, const EdgeScalars<T>& p, const DenseMatrix<T>& V);
template <typename T>
EdgeScalars<T> sddmm(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                     const SddmmKind& kind);
template <typename T>
std::pair<DenseMatrix<T>, DenseMatrix<T>> dense_oracle_forward(const Graph& g,
                                                               const DenseMatrix<T>& Q,
                                                               const DenseMatrix<T>& K,
                                                               const DenseMatrix<T>& V,
                                                               const SddmmKind& kind);

// --------------------------------------------------------------- autograd --
template <typename T>
struct GradBundle {
  DenseMatrix<T> dQ, dK, dV;
  /// Edge gradients: filled by the unfused schedule (unfused_backward, and
  /// fused_backward's infeasible-plan fallback); the fused recompute path
  /// never materialises E-sized tensors and leaves them empty.
  EdgeScalars<T> dS, dP;
};

/// Backward single steps (autograd.hpp:33-154), each a device op.
template <typename T>
std::pair<EdgeScalars<T>, DenseMatrix<T>> spmm_backward(const Graph& g, const EdgeScalars<T>& P,
                                                        const DenseMatrix<T>& V,
                                                        const DenseMatrix<T>& dO);
template <typename T>
EdgeScalars<T> softmax_backward(const Graph& g, const EdgeScalars<T>& P, const EdgeScalars<T>& dP);
template <typename T>
DenseMatrix<T> l2_normalize_backward(const DenseMatrix<T>& X, const DenseMatrix<T>& dY, T eps);
template <typename T>
std::pair<DenseMatrix<T>, DenseMatrix<T>> sddmm_backward(const Graph& g, const DenseMatrix<T>& Q,
                                                         const DenseMatrix<T>& K,
                                                         const EdgeScalars<T>& dS,
                                                         const SddmmKind& kind);

template <typename T>
struct BackwardResult {
  GradBundle<T> grads;
  ExecCounters counters;
};

namespace detail {
/// The unfused composition spmm_backward -> softmax_backward ->
/// sddmm_backward on the device (autograd.hpp:158-170), 5 launches, edge
/// gradients returned in dP / dS.  Uses ctx.P when it holds E values.
template <typename T>
GradBundle<T> backward_values(const Graph& g, const ForwardContext<T>& ctx,
                              const DenseMatrix<T>& dO);
template <typename T>
ExecCounters backward_counter_model(const Graph& g, const ForwardContext<T>& ctx,
                                    std::int64_t launches);
}  // namespace detail

template <typename T>
BackwardResult<T> unfused_backward(const Graph& g, const ForwardContext<T>& ctx,
                                   const DenseMatrix<T>& dO);
template <typename T>
BackwardResult<T> fused_backward(const Graph& g, const ForwardContext<T>& ctx,
                                 const DenseMatrix<T>& dO, const FusionPlan& plan);
/// Forward used by the finite-difference check (device forward, no P).
template <typename T>
DenseMatrix<T> reference_forward(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                                 const DenseMatrix<T>& V, const SddmmKind& kind);
template <typename T>
T finite_difference_check(const Graph& g, const DenseMatrix<T>& Q, const DenseMatrix<T>& K,
                          const DenseMatrix<T>& V, const SddmmKind& kind, T h);

// ----------------------------------------------------------------- models --
enum class Model { GT, AGNN, GAT };
std::string to_string(Model m);
Model model_from_string(const std::string& name);

struct ConvSpec {
  Model model = Model::GT;
  std::int64_t dim = 128;
  double scale = 0.0;
  double leaky_slope = 0.2;
  std::optional<Strategy> strategy_override;
};

SddmmKind kind_for(const ConvSpec& spec);

template <typename T>
struct ConvWeights {
  DenseMatrix<T> W_q, W_k, W_v;
  DenseMatrix<T> a_l, a_r;
};
template <typename T>
struct ConvContext {
  ForwardContext<T> fwd;
  DenseMatrix<T> X;
  DenseMatrix<T> H;
  ExecCounters counters;
};
template <typename T>
struct ConvGrads {
  GradBundle<T> pipeline;
  DenseMatrix<T> dW_q, dW_k, dW_v;
  DenseMatrix<T> da_l, da_r;
};

/// C = A * B and C = A^T * B on the device (gf_gemm).
template <typename T>
DenseMatrix<T> matmul(const DenseMatrix<T>& A, const DenseMatrix<T>& B);
template <typename T>
DenseMatrix<T> matmul_at_b(const DenseMatrix<T>& A, const DenseMatrix<T>& B);

template <typename T>
ConvWeights<T> random_weights(const ConvSpec& spec, std::int64_t d_in, std::uint64_t seed) {
  ConvWeights<T> w;
  const T lim = static_cast<T>(1.0 / std::sqrt(static_cast<double>(d_in)));
  w.W_v = random_matrix<T>(d_in, spec.dim, seed + 3, -lim, lim);
  if (spec.model == Model::GAT) {
    w.a_l = random_matrix<T>(spec.dim, 1, seed + 4, -lim, lim);
    w.a_r = random_matrix<T>(spec.dim, 1, seed + 5, -lim, lim);
  } else {
    w.W_q = random_matrix<T>(d_in, spec.dim, seed + 1, -lim, lim);
    w.W_k = random_matrix<T>(d_in, spec.dim, seed + 2, -lim, lim);
  }
  return w;
}

template <typename T>
std::pair<DenseMatrix<T>, ConvContext<T>> conv_forward(const ConvSpec& spec, const Graph& g,
                                                       const DenseMatrix<T>& X,
                                                       const ConvWeights<T>& w,
                                                       FusionPlan plan = FusionPlan{});
template <typename T>
ConvGrads<T> conv_backward(const ConvSpec& spec, const Graph& g, const ConvContext<T>& ctx,
                           const ConvWeights<T>& w, const DenseMatrix<T>& dO);

template <typename T>
struct PipelineInputs {
  DenseMatrix<T> Q, K, V;
  SddmmKind kind;
};
template <typename T>
PipelineInputs<T> make_pipeline_inputs(const Graph& g, const ConvSpec& spec, std::uint64_t seed);

double bandwidth_utilization(std::uint64_t bytes, double elapsed_s, double peak_bw_bytes_per_s);

}  // namespace graphfuse

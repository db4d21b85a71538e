// Planners (schedule.hpp:55-75 / schedule.cpp:26-88) and the modelled
// execution counters (counters.hpp:17-67, engine.hpp:84-168,
// autograd.hpp:172-190) of the drop-in API.  The counters are the
// reference's ANALYTIC model and are kept identical so the reference's
// counter tests hold unchanged; the B200 path's measured numbers (device
// time, ncu DRAM bytes) are reported separately (bench.py, profiles/).
#include <algorithm>
#include <stdexcept>

#include "graphfuse/graphfuse.hpp"

namespace graphfuse {

std::string to_string(Strategy s) {
  switch (s) {
    case Strategy::Smmf: return "smmf";
    case Strategy::Pmf: return "pmf";
    case Strategy::Unfused: return "unfused";
    case Strategy::FeatureParallelBaseline: return "baseline";
  }
  return "?";
}

Strategy strategy_from_string(const std::string& name) {
  static const std::pair<const char*, Strategy> table[] = {
      {"smmf", Strategy::Smmf},
      {"pmf", Strategy::Pmf},
      {"unfused", Strategy::Unfused},
      {"baseline", Strategy::FeatureParallelBaseline},
      {"feature-parallel", Strategy::FeatureParallelBaseline}};
  for (const auto& [k, v] : table)
    if (name == k) return v;
  throw std::invalid_argument("unknown strategy: " + name);
}

Strategy select_strategy(const DegreeStats& stats, const SddmmKind& kind,
                         std::int64_t shared_mem_bytes, std::int64_t dtype_bytes) {
  const bool dot = kind.variant == SddmmVariant::Dot;
  return dot && has_super_node(stats, shared_mem_bytes, dtype_bytes) ? Strategy::Pmf
                                                                     : Strategy::Smmf;
}

std::vector<RowRange> partition_blocks(const Graph& g, std::int64_t rows_per_block) {
  if (rows_per_block < 1)
    throw std::invalid_argument("partition_blocks: rows_per_block must be >= 1");
  std::vector<RowRange> out;
  out.reserve(static_cast<size_t>((g.num_nodes + rows_per_block - 1) / rows_per_block));
  for (NodeId v = 0; v < g.num_nodes; v += rows_per_block)
    out.push_back({v, std::min<NodeId>(g.num_nodes, v + rows_per_block)});
  return out;
}

namespace {
// Near-equal contiguous split of [lo, lo+total) into `parts` (first rem +1).
std::vector<EdgeRange> even_split(EdgeId lo, EdgeId total, std::int64_t parts) {
  std::vector<EdgeRange> out(static_cast<size_t>(parts));
  const EdgeId q = total / parts, r = total % parts;
  EdgeId at = lo;
  for (std::int64_t i = 0; i < parts; ++i) {
    const EdgeId len = q + (i < r ? 1 : 0);
    out[i] = {at, at + len};
    at += len;
  }
  return out;
}
}  // namespace

BlockAssignment warp_balance(const Graph& g, const RowRange& rows, std::int64_t groups_per_block) {
  if (groups_per_block < 1)
    throw std::invalid_argument("warp_balance: groups_per_block must be >= 1");
  BlockAssignment a;
  a.rows = rows;
  const EdgeId lo = g.csr_row_ptr[rows.begin];
  a.per_group_edges = even_split(lo, g.csr_row_ptr[rows.end] - lo, groups_per_block);
  return a;
}

std::vector<EdgeRange> edge_parallel_partition(const Graph& g, std::int64_t num_blocks) {
  if (num_blocks < 1)
    throw std::invalid_argument("edge_parallel_partition: num_blocks must be >= 1");
  if (g.num_edges == 0) return {};
  return even_split(0, g.num_edges, num_blocks);
}

std::int64_t shared_mem_usage(const FusionPlan& plan, std::int64_t block_max_edges,
                              std::int64_t d) {
  return plan.dtype_bytes * (2 * block_max_edges + plan.rows_per_block * d);
}

std::int64_t pmf_sddmm_block_count(const Graph& g, const FusionPlan& plan) {
  const std::int64_t per = std::max<std::int64_t>(1, plan.groups_per_block * plan.group_width);
  return std::max<std::int64_t>(1, (g.num_edges + per - 1) / per);
}

// ------------------------------------------------------------- counters --
std::uint64_t ExecCounters::max_group_load() const {
  std::uint64_t m = 0;
  for (auto x : per_group_edge_loads) m = std::max(m, x);
  return m;
}

double ExecCounters::mean_group_load() const {
  if (per_group_edge_loads.empty()) return 0.0;
  std::uint64_t t = 0;
  for (auto x : per_group_edge_loads) t += x;
  return static_cast<double>(t) / static_cast<double>(per_group_edge_loads.size());
}

std::map<std::string, std::uint64_t> ExecCounters::to_map(bool include_elapsed) const {
  std::map<std::string, std::uint64_t> m{
      {"global_bytes_read", global_bytes_read},
      {"global_bytes_written", global_bytes_written},
      {"shared_bytes_accessed", shared_bytes_accessed},
      {"memory_transactions", memory_transactions},
      {"kernel_launches", kernel_launches},
      {"softmax_scalar_ops", softmax_scalar_ops},
      {"s_global_bytes", s_global_bytes},
      {"f_global_bytes", f_global_bytes},
      {"p_global_bytes", p_global_bytes},
      {"max_group_load", max_group_load()},
      {"fallback_unfused", fallback_unfused ? 1u : 0u},
  };
  if (include_elapsed) m["elapsed_ns"] = elapsed_ns;
  return m;
}

bool ExecCounters::same_model(const ExecCounters& o) const {
  return per_group_edge_loads == o.per_group_edge_loads && to_map(false) == o.to_map(false);
}

namespace detail {

template <typename T>
ExecCounters model_counters(const Graph& g, const SddmmKind& kind, const FusionPlan& plan,
                            std::int64_t d, Strategy mode) {
  using U = std::uint64_t;
  const U b = sizeof(T), E = static_cast<U>(g.num_edges), N = static_cast<U>(g.num_nodes);
  const U dd = static_cast<U>(d), eb = E * b;
  const U sddmm_in = (kind.variant == SddmmVariant::Add ? 2 * b : 2 * dd * b) * E;
  const U tile = 2 * E * dd * b;  // output-tile accumulate, read + write per edge element
  // Redundancy-free softmax: 4 scalar ops (max, exp, sum, divide) per edge.
  U softmax_ops = 0;
  for (NodeId v = 0; v < g.num_nodes; ++v) softmax_ops += 4 * static_cast<U>(g.in_degree(v));

  ExecCounters c;
  c.memory_transactions = (E + N) * static_cast<U>(vectorized_transactions(d, plan.vector_width));
  c.global_bytes_read = sddmm_in + E * dd * b;
  c.global_bytes_written = N * dd * b;
  c.softmax_scalar_ops = softmax_ops;
  auto edge_parallel_loads = [&] {
    for (const auto& r : edge_parallel_partition(g, pmf_sddmm_block_count(g, plan)))
      c.per_group_edge_loads.push_back(static_cast<U>(r.size()));
  };
  switch (mode) {
    case Strategy::Unfused:
      c.kernel_launches = 3;
      c.s_global_bytes = c.f_global_bytes = c.p_global_bytes = 2 * eb;
      c.global_bytes_written += 3 * eb;
      c.global_bytes_read += 3 * eb;
      edge_parallel_loads();
      break;
    case Strategy::Smmf:
      c.kernel_launches = 1;
      c.p_global_bytes = eb;
      c.global_bytes_written += eb;
      c.shared_bytes_accessed = 5 * eb + tile;
      for (const auto& rows : partition_blocks(g, plan.rows_per_block))
        for (const auto& r : warp_balance(g, rows, plan.groups_per_block).per_group_edges)
          c.per_group_edge_loads.push_back(static_cast<U>(r.size()));
      break;
    case Strategy::Pmf:
      c.kernel_launches = 2;
      c.s_global_bytes = 2 * eb;
      c.p_global_bytes = eb;
      c.global_bytes_written += 2 * eb;
      c.global_bytes_read += eb;
      c.shared_bytes_accessed = 3 * eb + tile;
      edge_parallel_loads();
      break;
    case Strategy::FeatureParallelBaseline: {
      c.kernel_launches = 1;
      c.p_global_bytes = eb;
      c.global_bytes_written += eb;
      const U groups = static_cast<U>(
          std::max<std::int64_t>(1, (d + plan.group_width - 1) / plan.group_width));
      c.softmax_scalar_ops = groups * softmax_ops;
      c.shared_bytes_accessed = 2 * eb * groups + tile;
      c.per_group_edge_loads.reserve(N);
      for (NodeId v = 0; v < g.num_nodes; ++v)
        c.per_group_edge_loads.push_back(static_cast<U>(g.in_degree(v)));
      break;
    }
  }
  return c;
}

template <typename T>
void check_smmf_feasible(const Graph& g, const FusionPlan& plan, std::int64_t d) {
  FusionPlan p = plan;
  p.dtype_bytes = sizeof(T);
  const auto blocks = partition_blocks(g, plan.rows_per_block);
  for (size_t i = 0; i < blocks.size(); ++i) {
    const EdgeId edges = g.csr_row_ptr[blocks[i].end] - g.csr_row_ptr[blocks[i].begin];
    const std::int64_t need = shared_mem_usage(p, edges, d);
    if (need > plan.shared_mem_budget_bytes)
      throw EngineError("smmf infeasible: block " + std::to_string(i) + " requires " +
                        std::to_string(need) + " shared bytes, budget " +
                        std::to_string(plan.shared_mem_budget_bytes));
  }
}

template ExecCounters model_counters<float>(const Graph&, const SddmmKind&, const FusionPlan&,
                                            std::int64_t, Strategy);
template ExecCounters model_counters<double>(const Graph&, const SddmmKind&, const FusionPlan&,
                                             std::int64_t, Strategy);
template void check_smmf_feasible<float>(const Graph&, const FusionPlan&, std::int64_t);
template void check_smmf_feasible<double>(const Graph&, const FusionPlan&, std::int64_t);

}  // namespace detail

std::string to_string(Model m) {
  switch (m) {
    case Model::GT: return "gt";
    case Model::AGNN: return "agnn";
    case Model::GAT: return "gat";
  }
  return "?";
}

Model model_from_string(const std::string& name) {
  if (name == "gt") return Model::GT;
  if (name == "agnn") return Model::AGNN;
  if (name == "gat") return Model::GAT;
  throw std::invalid_argument("unknown model: " + name);
}

SddmmKind kind_for(const ConvSpec& spec) {
  switch (spec.model) {
    case Model::GT:  // scaled dot product, default 1/sqrt(dim)
      return SddmmKind::dot(spec.scale > 0 ? spec.scale
                                           : 1.0 / std::sqrt(static_cast<double>(spec.dim)));
    case Model::AGNN:  // cosine attention, beta defaults to 1
      return SddmmKind::dot(spec.scale > 0 ? spec.scale : 1.0, true);
    case Model::GAT:
      return SddmmKind::add(spec.leaky_slope);
  }
  throw std::invalid_argument("kind_for: bad model");
}

double bandwidth_utilization(std::uint64_t bytes, double elapsed_s, double peak_bw_bytes_per_s) {
  if (elapsed_s <= 0) throw std::invalid_argument("bandwidth_utilization: elapsed must be > 0");
  if (peak_bw_bytes_per_s <= 0)
    throw std::invalid_argument("bandwidth_utilization: peak bandwidth must be > 0");
  return static_cast<double>(bytes) / (elapsed_s * peak_bw_bytes_per_s);
}

}  // namespace graphfuse

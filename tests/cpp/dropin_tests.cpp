// C++ drop-in check: code written against the reference's operator API
// (#include "graphfuse/engine.hpp" etc., namespace graphfuse, templates on T)
// compiles unchanged against include/graphfuse and runs on the B200 path via
// libgraphfuse.so -> libgraphfuse_cuda.so.  The cases restate the reference's
// own unit tests (test_engine.cpp, test_autograd.cpp, test_models.cpp) with
// this file's own harness.  Exit code 0 = all checks passed.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>

#include "graphfuse/autograd.hpp"
#include "graphfuse/bench.hpp"
#include "graphfuse/engine.hpp"
#include "graphfuse/models.hpp"

using namespace graphfuse;

static int g_checks = 0, g_fail = 0;
#define EXPECT(cond)                                                             \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)

template <typename T>
static double floor1(const DenseMatrix<T>& a, const DenseMatrix<T>& b) {
  double w = 0;
  for (size_t i = 0; i < a.data.size(); ++i) {
    const double x = a.data[i], y = b.data[i];
    w = std::max(w, std::abs(x - y) / std::max({std::abs(x), std::abs(y), 1.0}));
  }
  return w;
}

// Dense masked reference of the single-head forward (independent of the API).
template <typename T>
static DenseMatrix<T> dense_forward(const Graph& g, const PipelineInputs<T>& in) {
  const auto& k = in.kind;
  DenseMatrix<T> O(g.num_nodes, in.V.cols);
  auto norm_rows = [](const DenseMatrix<T>& X) {
    DenseMatrix<T> Y = X;
    for (std::int64_t r = 0; r < X.rows; ++r) {
      double s = 0;
      for (std::int64_t c = 0; c < X.cols; ++c) s += double(X.at(r, c)) * X.at(r, c);
      const double n = std::max(std::sqrt(s), 1e-12);
      for (std::int64_t c = 0; c < X.cols; ++c) Y.at(r, c) = T(X.at(r, c) / n);
    }
    return Y;
  };
  const DenseMatrix<T> Q = k.l2_normalize_inputs ? norm_rows(in.Q) : in.Q;
  const DenseMatrix<T> K = k.l2_normalize_inputs ? norm_rows(in.K) : in.K;
  for (NodeId v = 0; v < g.num_nodes; ++v) {
    const EdgeId b = g.csr_row_ptr[v], e = g.csr_row_ptr[v + 1];
    if (b == e) continue;
    std::vector<double> s;
    for (EdgeId i = b; i < e; ++i) {
      const NodeId u = g.csr_col_idx[i];
      if (k.variant == SddmmVariant::Dot) {
        double d = 0;
        for (std::int64_t c = 0; c < Q.cols; ++c) d += double(Q.at(u, c)) * K.at(v, c);
        s.push_back(k.scale * d);
      } else {
        const double x = double(Q.data[u]) + K.data[v];
        s.push_back(x >= 0 ? x : k.leaky_slope * x);
      }
    }
    double m = s[0], z = 0;
    for (double x : s) m = std::max(m, x);
    for (double& x : s) z += (x = std::exp(x - m));
    for (std::int64_t c = 0; c < in.V.cols; ++c) {
      double acc = 0;
      for (EdgeId i = b; i < e; ++i) acc += s[i - b] / z * in.V.at(g.csr_col_idx[i], c);
      O.at(v, c) = T(acc);
    }
  }
  return O;
}

static void modes_match_dense() {
  for (std::uint64_t seed = 0; seed < 6; ++seed) {
    Graph g = gen_random(48 + seed * 30, 6, seed);
    ConvSpec spec;
    spec.model = seed % 3 == 0 ? Model::GT : seed % 3 == 1 ? Model::AGNN : Model::GAT;
    spec.dim = 8;
    auto in = make_pipeline_inputs<float>(g, spec, seed + 100);
    const auto ref = dense_forward(g, in);
    FusionPlan plan;
    for (Strategy m : {Strategy::Unfused, Strategy::Smmf, Strategy::Pmf,
                       Strategy::FeatureParallelBaseline}) {
      auto res = run_strategy(g, in.Q, in.K, in.V, in.kind, plan.with_strategy(m));
      EXPECT(floor1(res.O, ref) < 2e-5);
      EXPECT(res.ctx.P.size() == g.num_edges);
      for (NodeId v = 0; v < g.num_nodes; ++v) {
        double sum = 0;
        for (EdgeId i = g.csr_row_ptr[v]; i < g.csr_row_ptr[v + 1]; ++i) sum += res.ctx.P[i];
        if (g.in_degree(v) > 0) EXPECT(std::abs(sum - 1.0) < 1e-5);
      }
    }
  }
}

static void launches_and_traffic() {
  Graph g = gen_random(1000, 10, 5);
  EXPECT(g.num_edges == 10000);
  auto V = random_matrix<float>(1000, 4, 1), Q = random_matrix<float>(1000, 4, 2),
       K = random_matrix<float>(1000, 4, 3);
  FusionPlan plan;
  EXPECT(run_unfused(g, Q, K, V, SddmmKind::dot()).counters.kernel_launches == 3);
  EXPECT(run_pmf(g, Q, K, V, SddmmKind::dot(), plan).counters.kernel_launches == 2);
  EXPECT(run_smmf(g, Q, K, V, SddmmKind::dot(), plan).counters.kernel_launches == 1);
  const std::uint64_t eb = 10000 * 4;
  auto un = run_unfused(g, Q, K, V, SddmmKind::dot(), plan).counters;
  auto sm = run_smmf(g, Q, K, V, SddmmKind::dot(), plan).counters;
  EXPECT(un.s_global_bytes == 2 * eb && un.f_global_bytes == 2 * eb && un.p_global_bytes == 2 * eb);
  EXPECT(sm.s_global_bytes == 0 && sm.p_global_bytes == eb);
}

static void feasibility_error() {
  Graph g = gen_super_node(100, 2, 90, 1);
  auto V = random_matrix<float>(100, 8, 1);
  FusionPlan plan;
  plan.shared_mem_budget_bytes = 256;
  bool threw = false;
  try {
    run_smmf(g, V, V, V, SddmmKind::dot(), plan);
  } catch (const EngineError& e) {
    const std::string msg = e.what();
    threw = msg.find("block 0") != std::string::npos && msg.find("requires") != std::string::npos;
  }
  EXPECT(threw);
}

static void backward_cases() {
  // fused == unfused values, launches 3/5 (test_autograd.cpp "fused backward equals ...")
  for (std::uint64_t seed = 0; seed < 6; ++seed) {
    Graph g = gen_random(20 + seed * 40, 5, seed);
    ConvSpec spec;
    spec.model = seed % 3 == 0 ? Model::GT : seed % 3 == 1 ? Model::AGNN : Model::GAT;
    spec.dim = 5;
    auto in = make_pipeline_inputs<double>(g, spec, seed + 50);
    ForwardContext<double> ctx;
    ctx.g = &g;
    ctx.Q = in.Q;
    ctx.K = in.K;
    ctx.V = in.V;
    ctx.kind = in.kind;
    auto dO = random_matrix<double>(g.num_nodes, 5, seed + 60);
    auto f = fused_backward(g, ctx, dO, FusionPlan{});
    auto u = unfused_backward(g, ctx, dO);
    EXPECT(f.counters.kernel_launches == 3 && u.counters.kernel_launches == 5);
    EXPECT(!f.counters.fallback_unfused);
    EXPECT(floor1(f.grads.dQ, u.grads.dQ) < 1e-12 && floor1(f.grads.dV, u.grads.dV) < 1e-12);
  }
  // linearity in dO and zero dO (test_autograd.cpp)
  Graph g = gen_random(30, 4, 11);
  ConvSpec spec;
  spec.model = Model::GT;
  spec.dim = 3;
  auto in = make_pipeline_inputs<double>(g, spec, 12);
  auto res = run_strategy(g, in.Q, in.K, in.V, in.kind, FusionPlan{});
  auto dO = random_matrix<double>(30, 3, 13);
  auto one = unfused_backward(g, res.ctx, dO);
  for (double& v : dO.data) v *= -2.5;
  auto two = unfused_backward(g, res.ctx, dO);
  for (size_t i = 0; i < one.grads.dV.data.size(); ++i)
    EXPECT(std::abs(two.grads.dV.data[i] + 2.5 * one.grads.dV.data[i]) < 1e-10);
  auto zero = fused_backward(g, res.ctx, DenseMatrix<double>(30, 3), FusionPlan{});
  for (double v : zero.grads.dQ.data) EXPECT(v == 0.0);
  // finite differences (autograd.hpp:241-287) for all three models
  for (Model m : {Model::GT, Model::AGNN, Model::GAT}) {
    Graph gg = gen_random(12, 4, 21 + static_cast<int>(m));
    ConvSpec s;
    s.model = m;
    s.dim = 4;
    auto pin = make_pipeline_inputs<double>(gg, s, 22);
    EXPECT(finite_difference_check(gg, pin.Q, pin.K, pin.V, pin.kind, 1e-5) < 1e-6);
  }
}

static void layer_cases() {
  // GT with identity weights reduces to the raw pipeline (test_models.cpp)
  Graph g = gen_random(40, 4, 1);
  ConvSpec spec;
  spec.model = Model::GT;
  spec.dim = 8;
  auto X = random_matrix<double>(40, 8, 2);
  ConvWeights<double> w;
  w.W_q = w.W_k = w.W_v = DenseMatrix<double>(8, 8);
  for (int i = 0; i < 8; ++i) w.W_q.at(i, i) = w.W_k.at(i, i) = w.W_v.at(i, i) = 1;
  auto [O, ctx] = conv_forward(spec, g, X, w);
  FusionPlan plan;
  plan.strategy = ctx.fwd.plan.strategy;
  auto ref = run_strategy(g, X, X, X, kind_for(spec), plan);
  EXPECT(floor1(O, ref.O) < 1e-14);
  EXPECT(std::abs(ctx.fwd.kind.scale - 1.0 / std::sqrt(8.0)) < 1e-15);
  // conv_backward vs finite differences on W_v (GAT)
  ConvSpec gs;
  gs.model = Model::GAT;
  gs.dim = 3;
  auto Xg = random_matrix<double>(40, 4, 9);
  auto wg = random_weights<double>(gs, 4, 12);
  auto fw = conv_forward(gs, g, Xg, wg);
  auto grads = conv_backward(gs, g, fw.second, wg, DenseMatrix<double>(40, 3, 1.0));
  auto loss = [&](ConvWeights<double>& ww) {
    auto out = conv_forward(gs, g, Xg, ww).first;
    double s = 0;
    for (double v : out.data) s += v;
    return s;
  };
  for (size_t i = 0; i < wg.W_v.data.size(); i += 2) {
    const double keep = wg.W_v.data[i], h = 1e-6;
    wg.W_v.data[i] = keep + h;
    const double up = loss(wg);
    wg.W_v.data[i] = keep - h;
    const double dn = loss(wg);
    wg.W_v.data[i] = keep;
    const double fd = (up - dn) / (2 * h), a = grads.dW_v.data[i];
    EXPECT(std::abs(fd - a) / std::max({std::abs(fd), std::abs(a), 1.0}) < 1e-6);
  }
}

static bool near(double a, double b, double tol = 1e-12) {
  return std::abs(a - b) <= tol * std::max({std::abs(a), std::abs(b), 1.0});
}

// test_kernels.cpp:26-118 and test_autograd.cpp:28-158: the single-step
// operators, now device ops, on the reference's own known answers.
static void step_ops_cases() {
  Graph g = gen_random(16, 4, 3);
  DenseMatrix<double> ones(16, 2, 1.0);
  auto s1 = sddmm_dot(g, ones, ones, 1.0);
  bool ok = s1.size() == g.num_edges;
  for (EdgeId e = 0; e < g.num_edges; ++e) ok = ok && near(s1[e], 2.0);
  EXPECT(ok);
  Graph loops = from_coo(4, {0, 1, 2, 0}, {0, 1, 2, 1});
  DenseMatrix<double> Qd(4, 4);
  for (int i = 0; i < 4; ++i) Qd.at(i, i) = i + 1.0;
  auto so = sddmm_dot(loops, Qd, Qd, 2.0);
  EXPECT(near(so[0], 2.0) && near(so[1], 0.0) && near(so[2], 8.0) && near(so[3], 18.0));
  {
    auto Q = random_matrix<double>(16, 4, 1), K = random_matrix<double>(16, 4, 2);
    auto s = sddmm_dot(g, Q, K, 0.7);
    bool m = true;
    for (EdgeId e = 0; e < g.num_edges; ++e) {
      double acc = 0;
      for (int c = 0; c < 4; ++c) acc += Q.at(g.coo_src[e], c) * K.at(g.coo_dst[e], c);
      m = m && near(s[e], 0.7 * acc);
    }
    EXPECT(m);
  }
  bool threw = false;
  try {
    sddmm_dot(g, DenseMatrix<double>(16, 4), DenseMatrix<double>(16, 3), 1.0);
  } catch (const KernelError&) {
    threw = true;
  }
  EXPECT(threw);
  Graph one = from_coo(2, {0}, {1});
  DenseMatrix<double> el(2, 1), er(2, 1);
  el.data[0] = 1.0;
  er.data[1] = -3.0;
  EXPECT(near(sddmm_add(one, el, er, 0.2)[0], -0.4));
  DenseMatrix<double> X(1, 2);
  X.at(0, 0) = 3;
  X.at(0, 1) = 4;
  auto Y = l2_normalize_rows(X, 1e-12);
  EXPECT(near(Y.at(0, 0), 0.6) && near(Y.at(0, 1), 0.8));
  auto Z = l2_normalize_rows(DenseMatrix<double>(1, 3), 1e-12);
  EXPECT(Z.data[0] == 0.0 && Z.data[1] == 0.0 && Z.data[2] == 0.0);
  threw = false;
  try {
    l2_normalize_rows(DenseMatrix<double>(1, 1), 0.0);
  } catch (const KernelError&) {
    threw = true;
  }
  EXPECT(threw);
  // edge softmax: (0, 0) -> (1/2, 1/2); f32 (1000, 1001) -> (1/(1+e), e/(1+e))
  Graph two = from_coo(3, {0, 1}, {2, 2});
  EdgeScalars<float> sf(2);
  sf[0] = 1000.f;
  sf[1] = 1001.f;
  auto pf = edge_softmax(two, sf);
  EXPECT(std::abs(pf[0] - 1.0 / (1.0 + std::exp(1.0))) < 1e-5 &&
         std::abs(pf[1] - std::exp(1.0) / (1.0 + std::exp(1.0))) < 1e-5);
  // spmm: 1/2 weights give the mean; an empty row gives 0
  auto Vm = random_matrix<double>(3, 3, 4);
  auto Om = spmm(two, EdgeScalars<double>(2, 0.5), Vm);
  bool mean = true;
  for (int c = 0; c < 3; ++c)
    mean = mean && near(Om.at(2, c), 0.5 * (Vm.at(0, c) + Vm.at(1, c))) && Om.at(0, c) == 0.0;
  EXPECT(mean);
  // spmm_backward: identity P passes dO through; dense formulas on N=8
  {
    Graph id = from_coo(3, {0, 1, 2}, {0, 1, 2});
    auto V = random_matrix<double>(3, 4, 1), dO = random_matrix<double>(3, 4, 2);
    auto r = spmm_backward(id, EdgeScalars<double>(3, 1.0), V, dO);
    bool pass = true;
    for (size_t i = 0; i < r.second.data.size(); ++i) pass = pass && near(r.second.data[i], dO.data[i]);
    EXPECT(pass);
    Graph g8 = gen_random(8, 3, 3);
    auto V8 = random_matrix<double>(8, 3, 4), dO8 = random_matrix<double>(8, 3, 5);
    auto P8 = edge_softmax(g8, sddmm_dot(g8, V8, V8, 1.0));
    auto [dP, dV] = spmm_backward(g8, P8, V8, dO8);
    DenseMatrix<double> dVd(8, 3);
    bool dpok = true;
    for (EdgeId e = 0; e < g8.num_edges; ++e) {
      double acc = 0;
      for (int c = 0; c < 3; ++c) {
        acc += dO8.at(g8.coo_dst[e], c) * V8.at(g8.coo_src[e], c);
        dVd.at(g8.coo_src[e], c) += P8[e] * dO8.at(g8.coo_dst[e], c);
      }
      dpok = dpok && near(dP[e], acc);
    }
    EXPECT(dpok);
    EXPECT(floor1(dV, dVd) < 1e-12);
  }
  // softmax_backward: (1/2,1/2) with dP=(1,0) -> (1/4,-1/4); rows sum to zero
  {
    EdgeScalars<double> P(2, 0.5), dP(2);
    dP[0] = 1.0;
    auto dS = softmax_backward(two, P, dP);
    EXPECT(near(dS[0], 0.25) && near(dS[1], -0.25));
    Graph g50 = gen_random(50, 6, 8);
    auto sv = random_matrix<double>(g50.num_edges, 1, 9), dv = random_matrix<double>(g50.num_edges, 1, 10);
    EdgeScalars<double> S(g50.num_edges), dP2(g50.num_edges);
    S.values = sv.data;
    dP2.values = dv.data;
    auto dS2 = softmax_backward(g50, edge_softmax(g50, S), dP2);
    bool zero = true;
    for (NodeId v = 0; v < g50.num_nodes; ++v) {
      double sum = 0;
      for (EdgeId i = g50.csr_row_ptr[v]; i < g50.csr_row_ptr[v + 1]; ++i) sum += dS2[i];
      zero = zero && std::abs(sum) <= 1e-14 * std::max<EdgeId>(1, g50.csr_row_ptr[v + 1] - g50.csr_row_ptr[v]);
    }
    EXPECT(zero);
  }
  // sddmm_backward: single-edge product rule; dense dS K / dS^T Q
  {
    auto Q = random_matrix<double>(2, 3, 3), K = random_matrix<double>(2, 3, 4);
    auto [dQ, dK] = sddmm_backward(one, Q, K, EdgeScalars<double>(1, 1.0), SddmmKind::dot(1.0));
    bool pr = true;
    for (int c = 0; c < 3; ++c)
      pr = pr && near(dQ.at(0, c), K.at(1, c)) && near(dK.at(1, c), Q.at(0, c)) &&
           dQ.at(1, c) == 0.0 && dK.at(0, c) == 0.0;
    EXPECT(pr);
    Graph g9 = gen_random(9, 3, 5);
    auto Q9 = random_matrix<double>(9, 2, 6), K9 = random_matrix<double>(9, 2, 7);
    auto ds = random_matrix<double>(g9.num_edges, 1, 8);
    EdgeScalars<double> dS(g9.num_edges);
    dS.values = ds.data;
    auto [gq, gk] = sddmm_backward(g9, Q9, K9, dS, SddmmKind::dot(0.4));
    DenseMatrix<double> dq(9, 2), dk(9, 2);
    for (EdgeId e = 0; e < g9.num_edges; ++e)
      for (int c = 0; c < 2; ++c) {
        dq.at(g9.coo_src[e], c) += 0.4 * dS[e] * K9.at(g9.coo_dst[e], c);
        dk.at(g9.coo_dst[e], c) += 0.4 * dS[e] * Q9.at(g9.coo_src[e], c);
      }
    EXPECT(floor1(gq, dq) < 1e-12 && floor1(gk, dk) < 1e-12);
  }
  // fused == unfused (5 launches, edge gradients filled) for GT / AGNN / GAT
  for (std::uint64_t seed = 0; seed < 6; ++seed) {
    Graph gs = gen_random(20 + seed * 40, 5, seed);
    ConvSpec spec;
    spec.model = seed % 3 == 0 ? Model::GT : seed % 3 == 1 ? Model::AGNN : Model::GAT;
    spec.dim = 5;
    auto in = make_pipeline_inputs<double>(gs, spec, seed + 50);
    auto fr = run_strategy(gs, in.Q, in.K, in.V, in.kind, FusionPlan{});
    auto dO = random_matrix<double>(gs.num_nodes, 5, seed + 60);
    auto fb = fused_backward(gs, fr.ctx, dO, FusionPlan{});
    auto ub = unfused_backward(gs, fr.ctx, dO);
    EXPECT(fb.counters.kernel_launches == 3 && ub.counters.kernel_launches == 5);
    EXPECT(floor1(fb.grads.dQ, ub.grads.dQ) < 1e-11 && floor1(fb.grads.dK, ub.grads.dK) < 1e-11 &&
           floor1(fb.grads.dV, ub.grads.dV) < 1e-11);
    EXPECT(ub.grads.dP.size() == gs.num_edges && ub.grads.dS.size() == gs.num_edges);
  }
  // infeasible plan -> the unfused fallback (fills the edge gradients)
  {
    Graph gh = gen_super_node(100, 2, 90, 1);
    ConvSpec spec;
    spec.model = Model::GT;
    spec.dim = 4;
    auto in = make_pipeline_inputs<double>(gh, spec, 2);
    auto fr = run_strategy(gh, in.Q, in.K, in.V, in.kind, FusionPlan{});
    FusionPlan tight;
    tight.shared_mem_budget_bytes = 256;
    auto res = fused_backward(gh, fr.ctx, DenseMatrix<double>(100, 4, 1.0), tight);
    EXPECT(res.counters.fallback_unfused && res.counters.kernel_launches == 5);
    EXPECT(res.grads.dS.size() == gh.num_edges);
  }
}

// test_models.cpp:154-233 (benchmark runner, auto strategy, config parsing)
static void bench_cases() {
  BenchConfig cfg;
  cfg.model = "gt";
  cfg.nodes = 119;
  cfg.avg_degree = 12.0;
  cfg.batch_count = 4;
  cfg.dim = 32;
  cfg.seed = 3;
  cfg.strategies = {"auto", "unfused", "smmf", "pmf", "baseline"};
  cfg.peak_bw = 1.0e12;
  {
    BenchConfig bad = cfg;
    bad.peak_bw = 0.0;
    bool threw = false;
    try {
      run_benchmark(bad);
    } catch (const BenchError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  auto report = run_benchmark(cfg);
  EXPECT(report.num_nodes == 119 * 4);
  EXPECT(report.selected_strategy == "smmf");
  EXPECT(report.rows.size() == 4);
  EXPECT(report.rows[0].mode == "unfused");
  auto again = run_benchmark(cfg);
  for (size_t i = 0; i < report.rows.size() && i < again.rows.size(); ++i) {
    EXPECT(report.rows[i].mode == again.rows[i].mode);
    EXPECT(report.rows[i].counters.same_model(again.rows[i].counters));
    EXPECT(report.rows[i].device_ms > 0);  // every mode ran its own kernels
  }
  const std::string csv = report_csv(report);
  EXPECT(csv.rfind("mode,elapsed_ns,kernel_launches,global_bytes_read,"
                   "global_bytes_written,shared_bytes,memory_transactions,"
                   "softmax_scalar_ops,max_group_load,mean_group_load,"
                   "speedup_vs_unfused,bandwidth_utilization\n",
                   0) == 0);
  EXPECT(std::count(csv.begin(), csv.end(), '\n') == static_cast<long>(1 + report.rows.size()));
  EXPECT(report_markdown(report).find("| mode |") != std::string::npos);
  const std::string dcsv = report_csv_device(report);
  EXPECT(dcsv.find(",device_ms,device_speedup_vs_unfused,device_bandwidth_utilization,"
                   "device_dram_bytes\n") != std::string::npos);

  BenchConfig g = cfg;  // auto never picks PMF for additive attention
  g.model = "gat";
  g.nodes = 300;
  g.avg_degree = 2.0;
  g.hub_degree = 260;
  g.dim = 4;
  g.seed = 5;
  g.batch_count = 1;
  g.strategies = {"auto"};
  EXPECT(run_benchmark(g).selected_strategy != "pmf");

  BenchConfig p = config_from_json(R"({
    "model": "agnn", "nodes": 77, "avg_degree": 3.5, "dim": 16,
    "dtype": "f64", "seed": 9, "strategies": ["smmf", "unfused"],
    "deterministic": true, "peak_bw": 2.5e11
  })");
  EXPECT(p.model == "agnn" && p.nodes == 77 && p.avg_degree == 3.5 && p.dim == 16);
  EXPECT(p.dtype == "f64" && p.seed == 9 && p.strategies.size() == 2 && p.peak_bw == 2.5e11);
  bool bad_json = false;
  try {
    config_from_json("{not json");
  } catch (const BenchError&) {
    bad_json = true;
  }
  EXPECT(bad_json);
  auto r64 = run_benchmark(p);  // f64 agreement gate at 1e-11
  EXPECT(r64.rows.size() == 2);
}

int main() {
  modes_match_dense();
  launches_and_traffic();
  feasibility_error();
  backward_cases();
  layer_cases();
  step_ops_cases();
  bench_cases();
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}

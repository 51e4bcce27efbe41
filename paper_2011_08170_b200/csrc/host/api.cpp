// api.cpp — host C++ API (namespace f2m) over the C ABI of libf2m_gpu.so.
//
// Pure glue: type conversion, status -> exception mapping, lazy host views of device graphs.
// Every numeric routine of the solve path (k-NN, init, sweeps, dual objective, extraction,
// verification, jitter, restarts) executes on the GPU behind f2m_gpu.h.
#include <cmath>
#include <cstdio>
#include <mutex>
#include <ostream>
#include <sstream>

#include "f2m/api.hpp"
#include "f2m_gpu.h"

namespace f2m {
inline namespace b200 {

void throw_status(int status) {
  const std::string msg = f2m_last_error();
  switch (status) {
    case F2M_E_ARGUMENT: throw ArgumentError(msg);
    case F2M_E_INDEX: throw IndexError(msg);
    case F2M_E_MIN_DEGREE: throw MinDegreeError(msg);
    case F2M_E_STRUCTURE: throw StructureError(msg);
    case F2M_E_DEGREE: throw DegreeError(msg);
    case F2M_E_DEGENERATE: throw DegenerateExtraction(msg);
    case F2M_E_SOLVE_FAILED: throw SolveFailed(msg);
    default: throw DeviceError(msg.empty() ? "device failure" : msg);
  }
}

// ------------------------------------------------------------------ Graph

struct Graph::Impl {
  f2m_graph* h = nullptr;
  int n = 0;
  int64_t m = 0;
  double mean = 0.0;
  mutable std::once_flag edges_once, inc_once;
  mutable std::vector<GraphEdge> edges;
  mutable std::vector<int64_t> off;
  mutable std::vector<int> ids;
  explicit Impl(f2m_graph* handle) : h(handle) {
    f2m_graph_info info{};
    check(f2m_graph_get_info(h, &info));
    n = info.n;
    m = info.m;
    mean = info.mean_cost;
  }
  ~Impl() { f2m_graph_destroy(h); }
  void load_edges() const {
    std::call_once(edges_once, [&] {
      std::vector<int32_t> u(m), v(m);
      std::vector<double> c(m);
      check(f2m_graph_edges(h, u.data(), v.data(), c.data()));
      edges.resize(m);
      for (int64_t e = 0; e < m; ++e) edges[e] = GraphEdge{u[e], v[e], c[e]};
    });
  }
  void load_incidence() const {
    std::call_once(inc_once, [&] {
      off.assign(static_cast<size_t>(n) + 1, 0);
      std::vector<int32_t> tmp(static_cast<size_t>(2 * m) + 1);
      check(f2m_graph_incidence(h, off.data(), tmp.data()));
      ids.assign(tmp.begin(), tmp.begin() + off[n]);
    });
  }
};

Graph Graph::adopt(f2m_graph* handle) {
  Graph g;
  g.impl_ = std::make_shared<Impl>(handle);
  return g;
}

Graph Graph::from_edges(int n, std::vector<GraphEdge> edges) {
  if (n < 0) throw ArgumentError("from_edges: negative node count");
  const size_t m = edges.size();
  std::vector<int32_t> u(m), v(m);
  std::vector<double> c(m);
  for (size_t e = 0; e < m; ++e) {
    u[e] = edges[e].u;
    v[e] = edges[e].v;
    c[e] = edges[e].cost;
  }
  f2m_graph* h = nullptr;
  check(f2m_graph_from_edges(n, static_cast<int64_t>(m), u.data(), v.data(), c.data(), &h));
  return adopt(h);
}

int Graph::node_count() const { return impl_ ? impl_->n : 0; }
int Graph::edge_count() const { return impl_ ? static_cast<int>(impl_->m) : 0; }
double Graph::mean_cost() const { return impl_ ? impl_->mean : 0.0; }
f2m_graph* Graph::handle() const { return impl_ ? impl_->h : nullptr; }

const std::vector<GraphEdge>& Graph::edges() const {
  static const std::vector<GraphEdge> kEmpty;
  if (!impl_) return kEmpty;
  impl_->load_edges();
  return impl_->edges;
}

const GraphEdge& Graph::edge(int e) const { return edges()[static_cast<size_t>(e)]; }

std::span<const int> Graph::incident(int v) const {
  impl_->load_incidence();
  const auto& o = impl_->off;
  return std::span<const int>(impl_->ids.data() + o[v], impl_->ids.data() + o[v + 1]);
}

int Graph::degree(int v) const {
  if (!impl_) return 0;
  impl_->load_incidence();
  return static_cast<int>(impl_->off[v + 1] - impl_->off[v]);
}

int Graph::opposite(int e, int v) const {
  const GraphEdge& ge = edge(e);
  return ge.u == v ? ge.v : ge.u;
}

Graph Graph::with_costs(const std::vector<double>& costs) const {
  if (costs.size() != static_cast<size_t>(edge_count()))
    throw ArgumentError("with_costs: cost count does not match edge count");
  f2m_graph* h = nullptr;
  check(f2m_graph_with_costs(handle(), costs.data(), &h));
  return adopt(h);
}

static const Graph& need(const Graph& g) {
  if (!g.valid()) throw ArgumentError("graph is empty (default-constructed)");
  return g;
}

Graph build_knn_graph(const Instance& instance, int k, int /*threads*/) {
  const int n = instance.node_count();
  std::vector<double> xy(2 * static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    xy[2 * i] = instance.points[i].x;
    xy[2 * i + 1] = instance.points[i].y;
  }
  f2m_graph* h = nullptr;
  check(f2m_knn_build(n, xy.data(), instance.mode == DistanceMode::kEuc2dRounded ? 1 : 0, k, &h));
  return Graph::adopt(h);
}

GraphReport validate_graph(const Graph& graph) {
  GraphReport r;
  if (!graph.valid()) throw MinDegreeError("node degree 0 below 3; the node update needs a third-shortest edge");
  int mn = 0, mx = 0;
  int64_t m = 0;
  check(f2m_graph_validate(graph.handle(), &mn, &mx, &m));
  r.min_degree = mn;
  r.max_degree = mx;
  r.edge_count = static_cast<int>(m);
  return r;
}

void dump_edges(const Graph& graph, std::ostream& out) {
  char line[96];
  for (const GraphEdge& e : graph.edges()) {
    std::snprintf(line, sizeof(line), "%d %d %.17g\n", e.u, e.v, e.cost);
    out << line;
  }
}

// ------------------------------------------------------------------ dual engine

static f2m_engine_config to_c(const EngineConfig& c) {
  f2m_engine_config r{};
  r.b = c.b;
  r.eta = c.eta;
  r.eps = c.eps;
  r.max_sweeps = c.max_sweeps;
  r.mode = c.mode == SweepMode::kGaussSeidel ? 1 : 0;
  r.update = c.update == UpdateRule::kPaperDifference ? 1 : 0;
  r.init = c.init == DualInit::kZero ? 1 : 0;
  r.threads = c.threads;
  r.num_gpus = c.num_gpus;
  return r;
}

void EngineConfig::validate() const {
  const f2m_engine_config c = to_c(*this);
  check(f2m_engine_config_validate(&c));
}

static void check_size(const Graph& g, const DualState& s, const char* who) {
  if (s.lambda.size() != static_cast<size_t>(g.node_count()))
    throw ArgumentError(std::string(who) + ": state size does not match node count");
}

double adjusted_length(const Graph& graph, const DualState& state, int e) {
  if (e < 0 || e >= graph.edge_count()) throw IndexError("edge id out of range: " + std::to_string(e));
  const GraphEdge& ge = graph.edge(e);
  return ge.cost - state.lambda[static_cast<size_t>(ge.u)] - state.lambda[static_cast<size_t>(ge.v)];
}

double node_update_delta(const Graph& graph, const DualState& state, int v, int b) {
  need(graph);
  if (v < 0 || v >= graph.node_count()) throw IndexError("node id out of range: " + std::to_string(v));
  check_size(graph, state, "node_update_delta");
  double out = 0.0;
  check(f2m_node_update_delta(graph.handle(), state.lambda.data(), v, b, &out));
  return out;
}

std::vector<double> jacobi_sweeps(const Graph& graph, DualState& state, const EngineConfig& config,
                                  int count, double* dual_value) {
  config.validate();
  need(graph);
  check_size(graph, state, "jacobi_sweep");
  const f2m_engine_config c = to_c(config);
  std::vector<double> mx(static_cast<size_t>(std::max(count, 0)));
  check(f2m_jacobi_sweeps(graph.handle(), &c, state.lambda.data(), count, mx.data(), dual_value));
  return mx;
}

SweepStats jacobi_sweep(const Graph& graph, DualState& state, const EngineConfig& config) {
  SweepStats st;
  const std::vector<double> mx = jacobi_sweeps(graph, state, config, 1, &st.dual_value);
  st.max_abs_delta = mx[0];
  return st;
}

SweepStats jacobi_sweep(const Graph& graph, DualState& state, const EngineConfig& config, ThreadPool& /*pool*/,
                        std::vector<double>& delta_scratch) {
  config.validate();
  need(graph);
  check_size(graph, state, "jacobi_sweep");
  const f2m_engine_config c = to_c(config);
  delta_scratch.resize(static_cast<size_t>(graph.node_count()));
  if (graph.node_count() > 0) check(f2m_jacobi_deltas(graph.handle(), &c, state.lambda.data(), delta_scratch.data()));
  return jacobi_sweep(graph, state, config);
}

double dual_objective_pooled(const Graph& graph, const DualState& state, int b, ThreadPool* /*pool*/) {
  return dual_objective(graph, state, b);
}

SweepStats gauss_seidel_sweep(const Graph& graph, DualState& state, const EngineConfig& config) {
  config.validate();
  need(graph);
  check_size(graph, state, "gauss_seidel_sweep");
  const f2m_engine_config c = to_c(config);
  SweepStats st;
  check(f2m_gauss_seidel_sweeps(graph.handle(), &c, state.lambda.data(), 1, &st.max_abs_delta,
                                &st.dual_value));
  return st;
}

double dual_objective(const Graph& graph, const DualState& state, int b) {
  if (!graph.valid()) return 0.0;
  check_size(graph, state, "dual_objective");
  double out = 0.0;
  check(f2m_dual_objective(graph.handle(), state.lambda.data(), b, &out));
  return out;
}

std::pair<DualState, ConvergenceReport> solve_duals(const Graph& graph, const EngineConfig& config,
                                                    const std::optional<DualState>& initial) {
  config.validate();
  need(graph);
  if (initial.has_value() && initial->lambda.size() != static_cast<size_t>(graph.node_count()))
    throw ArgumentError("solve_duals: initial state size does not match node count");
  const f2m_engine_config c = to_c(config);
  DualState out;
  out.lambda.resize(static_cast<size_t>(graph.node_count()));
  f2m_convergence_report r{};
  check(f2m_solve_duals(graph.handle(), &c, initial ? initial->lambda.data() : nullptr, out.lambda.data(), &r));
  ConvergenceReport rep;
  rep.converged = r.converged != 0;
  rep.sweeps = r.sweeps;
  rep.final_max_abs_delta = r.final_max_abs_delta;
  rep.dual_value = r.dual_value;
  rep.wall_time = r.wall_time;
  return {std::move(out), rep};
}

DualState make_initial_state(const Graph& graph, const EngineConfig& config) {
  need(graph);
  const f2m_engine_config c = to_c(config);
  DualState s;
  s.lambda.resize(static_cast<size_t>(graph.node_count()));
  check(f2m_initial_state(graph.handle(), &c, s.lambda.data()));
  return s;
}

// ------------------------------------------------------------------ primal

EdgeClassification classify_edges(const Graph& graph, const DualState& state, double tol) {
  if (!(tol > 0.0)) throw ArgumentError("classify_edges: tol must be > 0");
  need(graph);
  check_size(graph, state, "classify_edges");
  std::vector<uint8_t> lab(static_cast<size_t>(graph.edge_count()));
  check(f2m_classify_edges(graph.handle(), state.lambda.data(), tol, lab.data()));
  EdgeClassification cls;
  cls.label.resize(lab.size());
  for (size_t e = 0; e < lab.size(); ++e) cls.label[e] = static_cast<EdgeSign>(lab[e]);
  return cls;
}

PrimalSolution extract_primal(const Graph& graph, const DualState& state, double tol) {
  need(graph);
  check_size(graph, state, "extract_primal");
  PrimalSolution sol;
  sol.value.resize(static_cast<size_t>(graph.edge_count()));
  check(f2m_extract_primal(graph.handle(), state.lambda.data(), tol, sol.value.data(), &sol.objective));
  return sol;
}

VerificationReport verify_solution(const Graph& graph, const PrimalSolution& solution,
                                   const DualState& state) {
  need(graph);
  check_size(graph, state, "verify_solution");
  if (solution.value.size() != static_cast<size_t>(graph.edge_count()))
    throw ArgumentError("verify_solution: solution size does not match edge count");
  const int64_t cap = std::max<int64_t>(graph.node_count(), graph.edge_count());
  std::vector<int32_t> nodes(static_cast<size_t>(cap) + 1), vals(static_cast<size_t>(cap) + 1);
  std::vector<double> sums(static_cast<size_t>(cap) + 1);
  f2m_verification r{};
  check(f2m_verify_solution(graph.handle(), solution.value.data(), solution.objective, state.lambda.data(), &r,
                            nodes.data(), sums.data(), vals.data(), cap));
  VerificationReport rep;
  rep.feasible = r.feasible != 0;
  rep.duality_gap = r.duality_gap;
  for (int64_t i = 0; i < r.violated_count; ++i) rep.violated_nodes.emplace_back(nodes[i], sums[i]);
  for (int64_t i = 0; i < r.value_violation_count; ++i) rep.value_violations.push_back(vals[i]);
  return rep;
}

void write_solution(const Graph& graph, const PrimalSolution& solution, const VerificationReport& report,
                    std::ostream& out) {
  char line[96];
  const auto& edges = graph.edges();
  for (size_t e = 0; e < edges.size(); ++e) {
    const double x = solution.value[e];
    if (x == 0.0) continue;
    std::snprintf(line, sizeof(line), "%d %d %g\n", edges[e].u, edges[e].v, x);
    out << line;
  }
  std::snprintf(line, sizeof(line), "objective %.17g gap %.17g\n", solution.objective, report.duality_gap);
  out << line;
}

std::vector<double> solve_zero_component(const Graph& graph, const std::vector<int>& component_edges,
                                         const std::vector<int>& residual) {
  need(graph);
  if (residual.size() < static_cast<size_t>(graph.node_count()))
    throw ArgumentError("solve_zero_component: residual must cover every node");
  std::vector<double> values(component_edges.size());
  int feasible = 0;
  check(f2m_solve_zero_component(graph.handle(), component_edges.data(), static_cast<int>(component_edges.size()),
                                 residual.data(), values.data(), &feasible));
  if (!feasible) values.clear();
  return values;
}

// ------------------------------------------------------------------ pipeline

static f2m_run_config to_c(const RunConfig& c) {
  f2m_run_config r{};
  r.k = c.k;
  r.engine = to_c(c.engine);
  r.tol = c.tol;
  r.gap_tol = c.gap_tol;
  r.max_restarts = c.max_restarts;
  r.perturb_scale = c.perturb_scale;
  r.seed = c.seed;
  return r;
}

double RunConfig::effective_tol() const { return tol > 0.0 ? tol : std::max(1e-7, 10.0 * engine.eps); }

void RunConfig::validate() const {
  const f2m_run_config c = to_c(*this);
  check(f2m_run_config_validate(&c));
}

SolveOutcome full_solve_graph(const Graph& graph, const RunConfig& config) {
  config.validate();
  if (!graph.valid()) throw MinDegreeError("node degree 0 below 3; the node update needs a third-shortest edge");
  const f2m_run_config c = to_c(config);
  SolveOutcome out;
  out.solution.value.resize(static_cast<size_t>(graph.edge_count()));
  out.duals.lambda.resize(static_cast<size_t>(graph.node_count()));
  f2m_solve_outcome r{};
  check(f2m_full_solve_graph(graph.handle(), &c, out.solution.value.data(), out.duals.lambda.data(), &r));
  out.solution.objective = r.objective;
  out.verification.feasible = r.verification.feasible != 0;
  out.verification.duality_gap = r.verification.duality_gap;
  out.convergence.converged = r.convergence.converged != 0;
  out.convergence.sweeps = r.convergence.sweeps;
  out.convergence.final_max_abs_delta = r.convergence.final_max_abs_delta;
  out.convergence.dual_value = r.convergence.dual_value;
  out.convergence.wall_time = r.convergence.wall_time;
  out.restarts = r.restarts;
  return out;
}

SolveOutcome full_solve(const Instance& instance, const RunConfig& config) {
  config.validate();
  const int k = std::min(config.k, instance.node_count() - 1);
  const Graph graph = build_knn_graph(instance, std::max(k, 3), config.engine.threads);
  return full_solve_graph(graph, config);
}

}  // namespace b200
}  // namespace f2m

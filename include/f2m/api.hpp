// f2m/api.hpp — host C++ surface of the B200-native solver.
//
// Same namespace (f2m), type names, function names, argument meaning and exception types as
// the reference's C++ API (/root/reference/proj/include/f2m/*.hpp), so code written against
// the reference compiles and behaves the same. Every compute call goes through the C ABI in
// f2m_gpu.h (hand-written sm_100a kernels); this layer only converts types and maps status
// codes onto exceptions. The inline namespace keeps the symbols distinct from the reference's
// own library when both are loaded in one process (the parity tests do that).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

struct f2m_graph;

namespace f2m {
inline namespace b200 {

// ------------------------------------------------------------------ exceptions (errors.hpp)
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ArgumentError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct IndexError : std::out_of_range { using std::out_of_range::out_of_range; };
struct MinDegreeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StructureError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegreeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegenerateExtraction : std::runtime_error { using std::runtime_error::runtime_error; };
struct TooLarge : std::runtime_error { using std::runtime_error::runtime_error; };
struct Infeasible : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolveFailed : std::runtime_error { using std::runtime_error::runtime_error; };
/// Device-side failure (no CUDA device, launch error, watchdog). Has no reference
/// counterpart: the reference never touches a GPU, and this solver never falls back to CPU.
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

/// Throws the f2m exception matching a C-ABI status (f2m_gpu.h) with f2m_last_error().
void throw_status(int status);
inline void check(int status) {
  if (status != 0) throw_status(status);
}

// ------------------------------------------------------------------ instances (instance.hpp)
struct Point {
  double x = 0.0;
  double y = 0.0;
};

enum class DistanceMode { kEuc2dRounded, kEuc2dExact };

struct Instance {
  std::string name;
  std::vector<Point> points;
  DistanceMode mode = DistanceMode::kEuc2dRounded;
  int node_count() const { return static_cast<int>(points.size()); }
};

Instance parse_tsplib(std::istream& in);
Instance parse_tsplib_string(const std::string& text);
Instance load_tsplib_file(const std::string& path);
void serialize_tsplib(const Instance& instance, std::ostream& out);
double distance(const Instance& instance, int i, int j);
Instance generate_instance(int n, std::uint64_t seed, double box = 1000.0);
/// Clustered synthetic instance (the reference has no clustered
/// generator): max(1, n/10) centres uniform in [0, box)^2 from one SplitMix64 stream, point i
/// = centre[i % centres] + N(0, box/sqrt(n))^2 by Box-Muller on the same stream. Exact mode.
Instance generate_clustered_instance(int n, std::uint64_t seed, double box = 1000.0);

struct SplitMix64 {
  std::uint64_t state = 0;
  explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// ------------------------------------------------------------------ graphs (graph.hpp)
struct GraphEdge {
  int u = 0;
  int v = 0;
  double cost = 0.0;
};

/// Immutable candidate graph, resident on the GPU. Host views (edges, incidence) are
/// downloaded lazily on first use and cached.
class Graph {
 public:
  Graph() = default;
  static Graph from_edges(int n, std::vector<GraphEdge> edges);
  /// Adopts a device graph handle created through the C ABI.
  static Graph adopt(f2m_graph* handle);

  int node_count() const;
  int edge_count() const;
  const GraphEdge& edge(int e) const;
  const std::vector<GraphEdge>& edges() const;
  std::span<const int> incident(int v) const;
  int degree(int v) const;
  int opposite(int e, int v) const;
  double mean_cost() const;
  Graph with_costs(const std::vector<double>& costs) const;

  /// The device handle (owned by this Graph and its copies).
  f2m_graph* handle() const;
  bool valid() const { return static_cast<bool>(impl_); }

 private:
  struct Impl;
  std::shared_ptr<Impl> impl_;
};

struct GraphReport {
  int min_degree = 0;
  int max_degree = 0;
  int edge_count = 0;
};

Graph build_knn_graph(const Instance& instance, int k, int threads = 0);
GraphReport validate_graph(const Graph& graph);
void dump_edges(const Graph& graph, std::ostream& out);

// ------------------------------------------------------------------ dual engine (dual.hpp)
struct DualState {
  std::vector<double> lambda;
};

enum class SweepMode { kJacobi, kGaussSeidel };
enum class UpdateRule { kMidpoint, kPaperDifference };
enum class DualInit { kLocalMidpoint, kZero };

struct EngineConfig {
  int b = 2;
  double eta = 0.5;
  double eps = 1e-9;
  int max_sweeps = 20000;
  SweepMode mode = SweepMode::kJacobi;
  UpdateRule update = UpdateRule::kMidpoint;
  DualInit init = DualInit::kLocalMidpoint;
  int threads = 0;  // accepted for compatibility; the device picks its own grid
  // B200 extension (f2m_engine_config.num_gpus): > 1 runs solve_duals' Jacobi sweeps on that many
  // GPUs from the calling thread (NVLink peer memory, one persistent kernel per GPU); bit-identical
  int num_gpus = 1;
  void validate() const;
};

struct SweepStats {
  double max_abs_delta = 0.0;
  double dual_value = 0.0;
  int sweep_index = 0;
};

struct ConvergenceReport {
  bool converged = false;
  int sweeps = 0;
  double final_max_abs_delta = 0.0;
  double dual_value = 0.0;
  double wall_time = 0.0;
};

double adjusted_length(const Graph& graph, const DualState& state, int e);
double node_update_delta(const Graph& graph, const DualState& state, int v, int b);
SweepStats jacobi_sweep(const Graph& graph, DualState& state, const EngineConfig& config);
SweepStats gauss_seidel_sweep(const Graph& graph, DualState& state, const EngineConfig& config);
double dual_objective(const Graph& graph, const DualState& state, int b = 2);
std::pair<DualState, ConvergenceReport> solve_duals(
    const Graph& graph, const EngineConfig& config,
    const std::optional<DualState>& initial = std::nullopt);
DualState make_initial_state(const Graph& graph, const EngineConfig& config);
// Internal entry points reusing a caller-owned pool (dual.hpp:83-87). The pool is accepted for
// source compatibility and not used: the sweep and the objective run on the GPU. delta_scratch
// receives every node's delta from the frozen snapshot, as the reference leaves it.
class ThreadPool;  // f2m/parallel.hpp
SweepStats jacobi_sweep(const Graph& graph, DualState& state, const EngineConfig& config, ThreadPool& pool,
                        std::vector<double>& delta_scratch);
double dual_objective_pooled(const Graph& graph, const DualState& state, int b, ThreadPool* pool);
/// `count` Jacobi sweeps in one persistent kernel; per-sweep max |delta| (B200 extension).
std::vector<double> jacobi_sweeps(const Graph& graph, DualState& state, const EngineConfig& config,
                                  int count, double* dual_value = nullptr);

// ------------------------------------------------------------------ primal (primal.hpp)
enum class EdgeSign : std::uint8_t { kNeg, kZero, kPos };

struct EdgeClassification {
  std::vector<EdgeSign> label;
};

struct PrimalSolution {
  std::vector<double> value;
  double objective = 0.0;
};

struct VerificationReport {
  bool feasible = false;
  std::vector<std::pair<int, double>> violated_nodes;
  double duality_gap = 0.0;
  std::vector<int> value_violations;
};

EdgeClassification classify_edges(const Graph& graph, const DualState& state, double tol);
PrimalSolution extract_primal(const Graph& graph, const DualState& state, double tol);
VerificationReport verify_solution(const Graph& graph, const PrimalSolution& solution,
                                   const DualState& state);
void write_solution(const Graph& graph, const PrimalSolution& solution,
                    const VerificationReport& report, std::ostream& out);
std::vector<double> solve_zero_component(const Graph& graph,
                                         const std::vector<int>& component_edges,
                                         const std::vector<int>& residual);

// ------------------------------------------------------------------ test oracle (oracle.hpp)
struct OracleResult {
  double optimum = 0.0;
  PrimalSolution solution;
  std::uint64_t enumerated = 0;
};
/// Exhaustive {0, 1/2, 1} enumeration (independent ground truth for tiny graphs; host code,
/// never used by the solver). Throws TooLarge / Infeasible.
OracleResult brute_force_f2m(const Graph& graph, int max_edges = 20);

// ------------------------------------------------------------------ pipeline (solve.hpp)
struct RunConfig {
  int k = 20;
  EngineConfig engine;
  double tol = 0.0;
  double gap_tol = 1e-6;
  int max_restarts = 5;
  double perturb_scale = 1e-7;
  std::uint64_t seed = 0;
  double effective_tol() const;
  void validate() const;
};

struct SolveOutcome {
  PrimalSolution solution;
  VerificationReport verification;
  ConvergenceReport convergence;
  DualState duals;
  int restarts = 0;
};

SolveOutcome full_solve(const Instance& instance, const RunConfig& config);
SolveOutcome full_solve_graph(const Graph& graph, const RunConfig& config);
void write_lp(const Graph& graph, std::ostream& out);

struct BenchRow {
  std::string instance;
  int nodes = 0;
  int edges = 0;
  int sweeps = 0;
  double seconds = 0.0;
  double gap = 0.0;
  int restarts = 0;
  bool ok = false;
  std::string error;
};

struct InstanceSource {
  std::string path;
  int synthetic_n = 0;
  std::uint64_t seed = 0;
  double box = 1000.0;
  static InstanceSource from_file(std::string p);
  static InstanceSource synthetic(int n, std::uint64_t seed, double box = 1000.0);
  Instance load() const;
  std::string id() const;
};

std::vector<BenchRow> run_benchmark(const std::vector<InstanceSource>& sources,
                                    const RunConfig& config);
void write_bench_csv(const std::vector<BenchRow>& rows, std::ostream& out);
void write_bench_json(const std::vector<BenchRow>& rows, std::ostream& out);

}  // namespace b200
}  // namespace f2m

// Reference-style C++ caller of the pooled internal entry points (dual.hpp:83-87) and
// f2m/parallel.hpp, compiled against include/f2m and linked to libf2m.so by
// tests/test_gpu_cpp_api.py. Prints one "ok ..." line per check; exits non-zero on a mismatch.
#include <cmath>
#include <cstdio>
#include <vector>

#include "f2m/dual.hpp"
#include "f2m/graph.hpp"
#include "f2m/instance.hpp"
#include "f2m/parallel.hpp"

using namespace f2m;

static int fails = 0;
static void expect(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "ok" : "FAIL", what);
  fails += ok ? 0 : 1;
}

int main() {
  const Instance inst = generate_instance(3000, 4, 1000.0);
  const Graph g = build_knn_graph(inst, 10);
  EngineConfig cfg;
  DualState a = make_initial_state(g, cfg), b = a;
  ThreadPool pool(4);
  std::vector<double> delta;
  const SweepStats sa = jacobi_sweep(g, a, cfg, pool, delta);
  const SweepStats sb = jacobi_sweep(g, b, cfg);
  expect(a.lambda == b.lambda, "pooled jacobi_sweep == jacobi_sweep (lambda)");
  expect(sa.max_abs_delta == sb.max_abs_delta && sa.dual_value == sb.dual_value, "pooled stats");
  expect(delta.size() == static_cast<size_t>(g.node_count()), "delta scratch sized n");
  // lambda_{k+1} = lambda_k + eta * delta (dual.cpp:156-160), max |delta| = the sweep's statistic
  DualState c = make_initial_state(g, cfg);
  double mx = 0.0;
  bool same = true;
  for (int v = 0; v < g.node_count(); ++v) {
    same = same && (c.lambda[v] + cfg.eta * delta[v] == a.lambda[v]);
    mx = std::max(mx, std::abs(delta[v]));
  }
  expect(same, "lambda + eta * delta_scratch reproduces the sweep");
  expect(mx == sa.max_abs_delta, "max |delta_scratch| == max_abs_delta");
  expect(dual_objective_pooled(g, a, 2, &pool) == dual_objective(g, a, 2), "dual_objective_pooled");
  expect(dual_objective_pooled(g, a, 2, nullptr) == dual_objective(g, a, 2), "dual_objective_pooled(nullptr)");
  // the pool itself: chunked ranges, deterministic chunk partials, exceptions rethrown
  std::vector<double> part(chunk_count(100000, kNodeChunk), 0.0);
  pool.for_chunks(100000, kNodeChunk, [&](std::int64_t ci, std::int64_t lo, std::int64_t hi) {
    double acc = 0.0;
    for (std::int64_t i = lo; i < hi; ++i) acc += 1.0 / (1.0 + static_cast<double>(i));
    part[ci] = acc;
  });
  ThreadPool one(1);
  std::vector<double> part1(part.size(), 0.0);
  one.for_chunks(100000, kNodeChunk, [&](std::int64_t ci, std::int64_t lo, std::int64_t hi) {
    double acc = 0.0;
    for (std::int64_t i = lo; i < hi; ++i) acc += 1.0 / (1.0 + static_cast<double>(i));
    part1[ci] = acc;
  });
  expect(combine_partials(part) == combine_partials(part1), "for_chunks deterministic across thread counts");
  bool threw = false;
  try {
    pool.for_chunks(10, 1, [](std::int64_t ci, std::int64_t, std::int64_t) {
      if (ci == 7) throw std::runtime_error("boom");
    });
  } catch (const std::runtime_error&) {
    threw = true;
  }
  expect(threw, "for_chunks rethrows the body's exception");
  EngineConfig two = cfg;
  two.b = 12;  // validate() rejects b > 8 (dual.cpp:70) before any device work
  bool arg = false;
  try {
    std::vector<double> d;
    DualState s = a;
    jacobi_sweep(g, s, two, pool, d);
  } catch (const ArgumentError&) {
    arg = true;
  }
  expect(arg, "pooled jacobi_sweep validates the config");
  std::printf("%s\n", fails ? "FAILED" : "ALL OK");
  return fails ? 1 : 0;
}

// enumerate.cpp — exhaustive F2M ground truth for tiny graphs (brute_force_f2m, the
// reference's test oracle, oracle.hpp:24). Host code by nature: exponential search over
// {0, 1/2, 1} per edge, used only to cross-check the GPU solver on <= ~45 edges.
//
// Search: edges in id order; per node a demand of 4 half-units; branch on 2, 1, 0 halves;
// prune when a node's demand exceeds twice its unassigned incident edges, and by an
// admissible bound (every open node buys its remaining halves from its cheapest unassigned
// edges at c/2 each; each edge is counted from both ends, hence the final halving).
#include <algorithm>
#include <cmath>
#include <limits>

#include "f2m/api.hpp"

namespace f2m {
inline namespace b200 {

namespace {

struct Search {
  int n = 0, m = 0;
  std::vector<int> a, b;
  std::vector<double> c;
  std::vector<std::vector<int>> inc_sorted;  // per node: incident edge ids by cost
  std::vector<int> need, open_edges, halves, best;
  double best_cost = std::numeric_limits<double>::infinity();
  std::uint64_t leaves = 0;

  double bound(int from) const {
    double total = 0.0;
    for (int v = 0; v < n; ++v) {
      int r = need[v];
      if (r == 0) continue;
      if (r > 2 * open_edges[v]) return std::numeric_limits<double>::infinity();
      for (int e : inc_sorted[v]) {
        if (e < from) continue;  // already assigned
        const int take = std::min(2, r);
        total += take * 0.5 * c[e];
        r -= take;
        if (r == 0) break;
      }
    }
    return 0.5 * total;
  }

  void run(int e, double acc) {
    if (acc + bound(e) >= best_cost) return;
    if (e == m) {
      ++leaves;
      best_cost = acc;
      best = halves;
      return;
    }
    --open_edges[a[e]];
    --open_edges[b[e]];
    for (int h = 2; h >= 0; --h) {
      if (h > need[a[e]] || h > need[b[e]]) continue;
      need[a[e]] -= h;
      need[b[e]] -= h;
      if (need[a[e]] <= 2 * open_edges[a[e]] && need[b[e]] <= 2 * open_edges[b[e]]) {
        halves[e] = h;
        run(e + 1, acc + 0.5 * h * c[e]);
        halves[e] = 0;
      }
      need[a[e]] += h;
      need[b[e]] += h;
    }
    ++open_edges[a[e]];
    ++open_edges[b[e]];
  }
};

}  // namespace

OracleResult brute_force_f2m(const Graph& graph, int max_edges) {
  const int m = graph.edge_count();
  if (m > max_edges)
    throw TooLarge("oracle limited to " + std::to_string(max_edges) + " edges, got " + std::to_string(m));
  Search s;
  s.n = graph.node_count();
  s.m = m;
  s.a.resize(m);
  s.b.resize(m);
  s.c.resize(m);
  s.inc_sorted.resize(s.n);
  s.need.assign(s.n, 4);
  s.open_edges.assign(s.n, 0);
  s.halves.assign(m, 0);
  for (int e = 0; e < m; ++e) {
    const GraphEdge& ge = graph.edge(e);
    s.a[e] = ge.u;
    s.b[e] = ge.v;
    s.c[e] = ge.cost;
    ++s.open_edges[ge.u];
    ++s.open_edges[ge.v];
    s.inc_sorted[ge.u].push_back(e);
    s.inc_sorted[ge.v].push_back(e);
  }
  for (auto& l : s.inc_sorted)
    std::sort(l.begin(), l.end(), [&](int x, int y) { return s.c[x] != s.c[y] ? s.c[x] < s.c[y] : x < y; });
  s.run(0, 0.0);
  if (!std::isfinite(s.best_cost)) throw Infeasible("no {0, 1/2, 1} assignment meets every degree-2 constraint");
  OracleResult r;
  r.enumerated = s.leaves;
  r.solution.value.resize(m);
  double obj = 0.0;
  for (int e = 0; e < m; ++e) {
    r.solution.value[e] = 0.5 * s.best[e];
    obj += s.c[e] * r.solution.value[e];
  }
  r.solution.objective = obj;
  r.optimum = obj;
  return r;
}

}  // namespace b200
}  // namespace f2m

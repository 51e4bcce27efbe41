// Golden-vector dumper over the UNMODIFIED reference library (oracle/_ref/libf2m_core.a).
//
// Test infrastructure only: it runs the reference's own public C++ API
// (generate_instance, build_knn_graph, make_initial_state, jacobi_sweep, solve_duals,
// extract_primal, verify_solution, full_solve_graph) single-threaded and writes every
// intermediate result the parity ladder compares, as raw little-endian
// arrays plus a JSON meta file, into an output directory. tests/golden/make_golden.py packs
// those into the committed fixtures.
//
// usage: f2m_dump OUT_DIR --synthetic N SEED BOX | --points FILE.f64 (x,y pairs)
//                 [--rounded] [--k K] [--sweeps S] [--eps E] [--max-sweeps M]
//                 [--init zero|local-midpoint] [--eta ETA] [--no-solve] [--seed JITTER_SEED]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "f2m/dual.hpp"
#include "f2m/errors.hpp"
#include "f2m/graph.hpp"
#include "f2m/instance.hpp"
#include "f2m/parallel.hpp"
#include "f2m/primal.hpp"
#include "f2m/solve.hpp"

using namespace f2m;

template <class T>
static void dump(const std::string& dir, const char* name, const std::vector<T>& v) {
  std::ofstream out(dir + "/" + name, std::ios::binary);
  out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: f2m_dump OUT_DIR --synthetic N SEED BOX | --points FILE ...\n");
    return 2;
  }
  const std::string dir = argv[1];
  Instance inst;
  int k = 10, sweeps = 0, max_sweeps = 20000;
  double eps = 1e-9, eta = 0.5;
  bool rounded = false, solve = true, full_only = false;
  std::uint64_t jitter_seed = 0;
  std::string init = "local-midpoint";
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--synthetic") {
      inst = generate_instance(std::atoi(argv[i + 1]), std::strtoull(argv[i + 2], nullptr, 10),
                               std::atof(argv[i + 3]));
      i += 3;
    } else if (a == "--points") {
      std::ifstream in(argv[++i], std::ios::binary);
      std::vector<char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
      const std::size_t npts = buf.size() / 16;
      inst.points.resize(npts);
      std::memcpy(inst.points.data(), buf.data(), npts * 16);
      inst.mode = DistanceMode::kEuc2dExact;
      inst.name = "points";
    } else if (a == "--rounded") {
      rounded = true;
    } else if (a == "--k") {
      k = std::atoi(argv[++i]);
    } else if (a == "--sweeps") {
      sweeps = std::atoi(argv[++i]);
    } else if (a == "--eps") {
      eps = std::atof(argv[++i]);
    } else if (a == "--eta") {
      eta = std::atof(argv[++i]);
    } else if (a == "--max-sweeps") {
      max_sweeps = std::atoi(argv[++i]);
    } else if (a == "--init") {
      init = argv[++i];
    } else if (a == "--no-solve") {
      solve = false;
    } else if (a == "--full-only") {
      full_only = true;
    } else if (a == "--seed") {
      jitter_seed = std::strtoull(argv[++i], nullptr, 10);
    } else {
      std::fprintf(stderr, "unknown arg %s\n", a.c_str());
      return 2;
    }
  }
  if (rounded) inst.mode = DistanceMode::kEuc2dRounded;
  const int n = inst.node_count();
  std::vector<double> xy;
  for (const auto& p : inst.points) {
    xy.push_back(p.x);
    xy.push_back(p.y);
  }
  dump(dir, "points.f64", xy);

  double t0 = now();
  const Graph g = build_knn_graph(inst, std::max(3, std::min(k, n - 1)), 1);
  const double t_knn = now() - t0;
  std::vector<int> eu, ev;
  std::vector<double> ec;
  for (const auto& e : g.edges()) {
    eu.push_back(e.u);
    ev.push_back(e.v);
    ec.push_back(e.cost);
  }
  dump(dir, "eu.i32", eu);
  dump(dir, "ev.i32", ev);
  dump(dir, "ec.f64", ec);

  EngineConfig cfg;
  cfg.threads = 1;
  cfg.eps = eps;
  cfg.eta = eta;
  cfg.max_sweeps = max_sweeps;
  cfg.init = init == "zero" ? DualInit::kZero : DualInit::kLocalMidpoint;

  DualState st = make_initial_state(g, cfg);
  dump(dir, "lam0.f64", st.lambda);
  std::vector<double> stats;  // (max_abs_delta, dual_value) per sweep
  {
    ThreadPool pool(1);
    std::vector<double> scratch;
    for (int s = 0; s < sweeps; ++s) {
      SweepStats ss = jacobi_sweep(g, st, cfg, pool, scratch);
      stats.push_back(ss.max_abs_delta);
      stats.push_back(ss.dual_value);
    }
  }
  dump(dir, "lamN.f64", st.lambda);
  dump(dir, "sweep_stats.f64", stats);

  FILE* meta = std::fopen((dir + "/meta.json").c_str(), "w");
  std::fprintf(meta, "{\"n\": %d, \"m\": %d, \"k\": %d, \"rounded\": %d, \"mean_cost\": %.17g, "
               "\"sweeps_dumped\": %d, \"eps\": %.17g, \"eta\": %.17g, \"init\": \"%s\", "
               "\"max_sweeps\": %d, \"t_knn\": %.6f",
               n, g.edge_count(), k, rounded ? 1 : 0, g.mean_cost(), sweeps, eps, eta, init.c_str(),
               max_sweeps, t_knn);
  if (solve && full_only) {
    RunConfig rc;
    rc.k = k;
    rc.engine = cfg;
    rc.seed = jitter_seed;
    t0 = now();
    SolveOutcome out = full_solve_graph(g, rc);
    const double t_full = now() - t0;
    dump(dir, "x_full.f64", out.solution.value);
    dump(dir, "lam_full.f64", out.duals.lambda);
    std::fprintf(meta, ", \"full_ok\": 1, \"full_objective\": %.17g, \"full_gap\": %.17g, "
                 "\"full_restarts\": %d, \"full_sweeps\": %d, \"full_feasible\": %d, \"t_full\": %.6f, "
                 "\"sweeps\": %d, \"dual_value\": %.17g, \"final_max_abs_delta\": %.17g, \"converged\": %d",
                 out.solution.objective, out.verification.duality_gap, out.restarts, out.convergence.sweeps,
                 out.verification.feasible ? 1 : 0, t_full, out.convergence.sweeps, out.convergence.dual_value,
                 out.convergence.final_max_abs_delta, out.convergence.converged ? 1 : 0);
  } else if (solve) {
    t0 = now();
    auto [lam, rep] = solve_duals(g, cfg);
    const double t_solve = now() - t0;
    dump(dir, "lam_final.f64", lam.lambda);
    std::fprintf(meta, ", \"converged\": %d, \"sweeps\": %d, \"final_max_abs_delta\": %.17g, "
                 "\"dual_value\": %.17g, \"t_solve\": %.6f",
                 rep.converged ? 1 : 0, rep.sweeps, rep.final_max_abs_delta, rep.dual_value, t_solve);
    RunConfig rc;
    rc.k = k;
    rc.engine = cfg;
    rc.seed = jitter_seed;
    const double tol = rc.effective_tol() * (g.mean_cost() > 0.0 ? g.mean_cost() : 1.0);
    try {
      t0 = now();
      PrimalSolution sol = extract_primal(g, lam, tol);
      VerificationReport vr = verify_solution(g, sol, lam);
      const double t_ext = now() - t0;
      dump(dir, "x.f64", sol.value);
      std::fprintf(meta, ", \"extract_ok\": 1, \"objective\": %.17g, \"feasible\": %d, "
                   "\"gap\": %.17g, \"t_extract\": %.6f",
                   sol.objective, vr.feasible ? 1 : 0, vr.duality_gap, t_ext);
    } catch (const std::exception& e) {
      std::fprintf(meta, ", \"extract_ok\": 0");
    }
    try {
      t0 = now();
      SolveOutcome out = full_solve_graph(g, rc);
      const double t_full = now() - t0;
      dump(dir, "x_full.f64", out.solution.value);
      dump(dir, "lam_full.f64", out.duals.lambda);
      std::fprintf(meta, ", \"full_ok\": 1, \"full_objective\": %.17g, \"full_gap\": %.17g, "
                   "\"full_restarts\": %d, \"full_sweeps\": %d, \"full_feasible\": %d, \"t_full\": %.6f",
                   out.solution.objective, out.verification.duality_gap, out.restarts,
                   out.convergence.sweeps, out.verification.feasible ? 1 : 0, t_full);
    } catch (const std::exception& e) {
      std::fprintf(meta, ", \"full_ok\": 0");
    }
  }
  std::fprintf(meta, "}\n");
  std::fclose(meta);
  return 0;
}

// bindings.cpp — pybind11 module `_f2m`: the reference's Python surface
// (/root/reference/proj/python/bindings.cpp — same function names, keyword arguments, defaults
// and exception mapping) over the B200 solver, plus numpy/device entry points used by the
// benchmark and the parity tests.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <sstream>

#include "f2m/api.hpp"
#include "f2m_gpu.h"

namespace py = pybind11;

namespace {

f2m::EngineConfig engine_config(int b, double eta, double eps, int max_sweeps, const std::string& mode,
                                const std::string& update, const std::string& init, int threads) {
  f2m::EngineConfig c;
  c.b = b;
  c.eta = eta;
  c.eps = eps;
  c.max_sweeps = max_sweeps;
  c.mode = mode == "gauss-seidel" ? f2m::SweepMode::kGaussSeidel : f2m::SweepMode::kJacobi;
  c.update = update == "paper-difference" ? f2m::UpdateRule::kPaperDifference : f2m::UpdateRule::kMidpoint;
  c.init = init == "zero" ? f2m::DualInit::kZero : f2m::DualInit::kLocalMidpoint;
  c.threads = threads;
  c.validate();
  return c;
}

f2m_run_config run_config_c(int k, double eta, double eps, int max_sweeps, const std::string& mode, double tol,
                            int max_restarts, std::uint64_t seed, double gap_tol, double perturb_scale) {
  f2m_run_config rc{};
  rc.k = k;
  rc.engine.b = 2;
  rc.engine.eta = eta;
  rc.engine.eps = eps;
  rc.engine.max_sweeps = max_sweeps;
  rc.engine.mode = mode == "gauss-seidel" ? 1 : 0;
  rc.tol = tol;
  rc.gap_tol = gap_tol;
  rc.max_restarts = max_restarts;
  rc.perturb_scale = perturb_scale;
  rc.seed = seed;
  return rc;
}

py::dict outcome_dict(const f2m_solve_outcome& o) {
  return py::dict(py::arg("objective") = o.objective, py::arg("feasible") = o.verification.feasible != 0,
                  py::arg("gap") = o.verification.duality_gap, py::arg("sweeps") = o.convergence.sweeps,
                  py::arg("converged") = o.convergence.converged != 0,
                  py::arg("final_max_abs_delta") = o.convergence.final_max_abs_delta,
                  py::arg("dual_value") = o.convergence.dual_value, py::arg("restarts") = o.restarts,
                  py::arg("t_knn") = o.t_knn, py::arg("t_duals") = o.t_duals, py::arg("t_extract") = o.t_extract,
                  py::arg("t_total") = o.t_total);
}

}  // namespace

PYBIND11_MODULE(_f2m, m) {
  m.doc() = "B200-native fractional 2-matching solver (GDP over k-NN graphs, sm_100a)";

  py::register_exception<f2m::ParseError>(m, "ParseError", PyExc_ValueError);
  py::register_exception<f2m::DegenerateExtraction>(m, "DegenerateExtraction", PyExc_RuntimeError);
  py::register_exception<f2m::TooLarge>(m, "TooLarge", PyExc_ValueError);
  py::register_exception<f2m::Infeasible>(m, "Infeasible", PyExc_RuntimeError);
  py::register_exception<f2m::SolveFailed>(m, "SolveFailed", PyExc_RuntimeError);
  py::register_exception<f2m::DeviceError>(m, "DeviceError", PyExc_RuntimeError);

  py::enum_<f2m::DistanceMode>(m, "DistanceMode")
      .value("EUC2D_ROUNDED", f2m::DistanceMode::kEuc2dRounded)
      .value("EUC2D_EXACT", f2m::DistanceMode::kEuc2dExact);

  py::class_<f2m::Instance>(m, "Instance")
      .def_readonly("name", &f2m::Instance::name)
      .def_readwrite("mode", &f2m::Instance::mode)
      .def_property_readonly("points",
                             [](const f2m::Instance& inst) {
                               std::vector<std::pair<double, double>> pts;
                               pts.reserve(inst.points.size());
                               for (const auto& p : inst.points) pts.emplace_back(p.x, p.y);
                               return pts;
                             })
      .def("__len__", &f2m::Instance::node_count)
      .def("distance", [](const f2m::Instance& inst, int i, int j) { return f2m::distance(inst, i, j); })
      // --- extensions: zero-copy-ish numpy construction and export
      .def_static(
          "from_points",
          [](py::array_t<double, py::array::c_style | py::array::forcecast> xy, f2m::DistanceMode mode,
             const std::string& name) {
            if (xy.ndim() != 2 || xy.shape(1) != 2) throw f2m::ArgumentError("from_points: expected an (n, 2) array");
            f2m::Instance inst;
            inst.name = name;
            inst.mode = mode;
            inst.points.resize(static_cast<size_t>(xy.shape(0)));
            const double* p = xy.data();
            for (size_t i = 0; i < inst.points.size(); ++i) inst.points[i] = f2m::Point{p[2 * i], p[2 * i + 1]};
            return inst;
          },
          py::arg("xy"), py::arg("mode") = f2m::DistanceMode::kEuc2dExact, py::arg("name") = "")
      .def("points_array", [](const f2m::Instance& inst) {
        py::array_t<double> a({static_cast<py::ssize_t>(inst.points.size()), static_cast<py::ssize_t>(2)});
        double* p = a.mutable_data();
        for (size_t i = 0; i < inst.points.size(); ++i) {
          p[2 * i] = inst.points[i].x;
          p[2 * i + 1] = inst.points[i].y;
        }
        return a;
      });

  m.def("parse_tsplib", &f2m::parse_tsplib_string, py::arg("text"));
  m.def("load_tsplib", &f2m::load_tsplib_file, py::arg("path"));
  m.def(
      "serialize_tsplib",
      [](const f2m::Instance& instance) {
        std::ostringstream out;
        f2m::serialize_tsplib(instance, out);
        return out.str();
      },
      py::arg("instance"));
  m.def("generate_instance", &f2m::generate_instance, py::arg("n"), py::arg("seed"), py::arg("box") = 1000.0);
  m.def("generate_clustered_instance", &f2m::generate_clustered_instance, py::arg("n"), py::arg("seed"),
        py::arg("box") = 1000.0);

  py::class_<f2m::Graph>(m, "Graph")
      .def_property_readonly("n", &f2m::Graph::node_count)
      .def_property_readonly("m", &f2m::Graph::edge_count)
      .def("edges",
           [](const f2m::Graph& g) {
             std::vector<std::tuple<int, int, double>> out;
             out.reserve(g.edges().size());
             for (const auto& e : g.edges()) out.emplace_back(e.u, e.v, e.cost);
             return out;
           })
      .def("degree", &f2m::Graph::degree)
      .def("mean_cost", &f2m::Graph::mean_cost)
      // --- extensions
      .def("edge_arrays",
           [](const f2m::Graph& g) {
             const py::ssize_t mm = g.edge_count();
             py::array_t<int32_t> u(mm), v(mm);
             py::array_t<double> c(mm);
             if (mm) f2m::check(f2m_graph_edges(g.handle(), u.mutable_data(), v.mutable_data(), c.mutable_data()));
             return py::make_tuple(u, v, c);
           })
      .def("positions",
           [](const f2m::Graph& g) {
             py::array_t<int32_t> p(g.node_count());
             if (g.node_count()) f2m::check(f2m_graph_positions(g.handle(), p.mutable_data()));
             return p;
           })
      .def("degrees",
           [](const f2m::Graph& g) {
             py::array_t<int32_t> d(g.node_count());
             if (g.node_count()) f2m::check(f2m_graph_degrees(g.handle(), d.mutable_data()));
             return d;
           })
      .def("with_costs", &f2m::Graph::with_costs, py::arg("costs"))
      .def("sell_slots",
           [](const f2m::Graph& g) {
             f2m_graph_info info{};
             f2m::check(f2m_graph_get_info(g.handle(), &info));
             return info.sell_slots;
           })
      .def("sweep_bytes", [](const f2m::Graph& g) { return f2m_sweep_algorithmic_bytes(g.handle()); })
      .def("layout", [](const f2m::Graph& g) {
        f2m_graph_info i{};
        f2m::check(f2m_graph_get_info(g.handle(), &i));
        return py::dict(py::arg("n") = i.n, py::arg("m") = i.m, py::arg("sell_slots") = i.sell_slots,
                        py::arg("min_degree") = i.min_degree, py::arg("max_degree") = i.max_degree,
                        py::arg("sweep_ctas") = i.sweep_ctas, py::arg("sweep_variant") = i.sweep_variant,
                        py::arg("max_local") = i.max_local, py::arg("max_cta_slots") = i.max_cta_slots,
                        py::arg("smem_bytes") = i.smem_bytes);
      });

  m.def(
      "build_knn_graph",
      [](const f2m::Instance& instance, int k, int threads) { return f2m::build_knn_graph(instance, k, threads); },
      py::arg("instance"), py::arg("k"), py::arg("threads") = 0, py::call_guard<py::gil_scoped_release>());
  m.def(
      "graph_from_edges",
      [](int n, py::array_t<int32_t, py::array::c_style | py::array::forcecast> u,
         py::array_t<int32_t, py::array::c_style | py::array::forcecast> v,
         py::array_t<double, py::array::c_style | py::array::forcecast> c) {
        if (u.size() != v.size() || u.size() != c.size()) throw f2m::ArgumentError("graph_from_edges: length mismatch");
        f2m_graph* h = nullptr;
        f2m::check(f2m_graph_from_edges(n, u.size(), u.data(), v.data(), c.data(), &h));
        return f2m::Graph::adopt(h);
      },
      py::arg("n"), py::arg("u"), py::arg("v"), py::arg("cost"));
  m.def("validate_graph", [](const f2m::Graph& g) {
    const f2m::GraphReport r = f2m::validate_graph(g);
    return py::dict(py::arg("min_degree") = r.min_degree, py::arg("max_degree") = r.max_degree,
                    py::arg("edge_count") = r.edge_count);
  });

  py::class_<f2m::DualState>(m, "DualState")
      .def(py::init<>())
      .def(py::init([](std::vector<double> lam) { return f2m::DualState{std::move(lam)}; }), py::arg("lam"))
      .def_readwrite("lam", &f2m::DualState::lambda);

  m.def("dual_objective", &f2m::dual_objective, py::arg("graph"), py::arg("state"), py::arg("b") = 2);
  m.def("adjusted_length", &f2m::adjusted_length, py::arg("graph"), py::arg("state"), py::arg("edge"));
  m.def("node_update_delta", &f2m::node_update_delta, py::arg("graph"), py::arg("state"), py::arg("node"),
        py::arg("b") = 2);

  m.def(
      "solve_duals",
      [](const f2m::Graph& graph, int b, double eta, double eps, int max_sweeps, const std::string& mode,
         const std::string& update, const std::string& init, int threads, std::optional<f2m::DualState> initial,
         int num_gpus) {
        f2m::EngineConfig config = engine_config(b, eta, eps, max_sweeps, mode, update, init, threads);
        config.num_gpus = num_gpus;
        std::pair<f2m::DualState, f2m::ConvergenceReport> res;
        {
          py::gil_scoped_release release;
          res = f2m::solve_duals(graph, config, initial);
        }
        const auto& r = res.second;
        py::dict rep(py::arg("converged") = r.converged, py::arg("sweeps") = r.sweeps,
                     py::arg("final_max_abs_delta") = r.final_max_abs_delta, py::arg("dual_value") = r.dual_value,
                     py::arg("wall_time") = r.wall_time);
        return py::make_tuple(res.first, rep);
      },
      py::arg("graph"), py::arg("b") = 2, py::arg("eta") = 0.5, py::arg("eps") = 1e-9, py::arg("max_sweeps") = 20000,
      py::arg("mode") = "jacobi", py::arg("update") = "midpoint", py::arg("init") = "local-midpoint",
      py::arg("threads") = 0, py::arg("initial") = py::none(), py::arg("num_gpus") = 1);

  // --- extensions: the sweep-level entry points the reference keeps C++-only (dual.hpp:66-90)
  m.def(
      "make_initial_state",
      [](const f2m::Graph& graph, int b, const std::string& init) {
        return f2m::make_initial_state(graph, engine_config(b, 0.5, 1e-9, 0, "jacobi", "midpoint", init, 0));
      },
      py::arg("graph"), py::arg("b") = 2, py::arg("init") = "local-midpoint");
  m.def(
      "jacobi_sweeps",
      [](const f2m::Graph& graph, f2m::DualState& state, int count, int b, double eta, const std::string& update) {
        const f2m::EngineConfig c = engine_config(b, eta, 1e-9, 0, "jacobi", update, "local-midpoint", 0);
        double dv = 0.0;
        std::vector<double> mx;
        {
          py::gil_scoped_release release;
          mx = f2m::jacobi_sweeps(graph, state, c, count, &dv);
        }
        return py::make_tuple(mx, dv);
      },
      py::arg("graph"), py::arg("state"), py::arg("count"), py::arg("b") = 2, py::arg("eta") = 0.5,
      py::arg("update") = "midpoint");
  m.def(
      "jacobi_sweep",
      [](const f2m::Graph& graph, f2m::DualState& state, int b, double eta, const std::string& update) {
        const f2m::SweepStats s =
            f2m::jacobi_sweep(graph, state, engine_config(b, eta, 1e-9, 0, "jacobi", update, "local-midpoint", 0));
        return py::make_tuple(s.max_abs_delta, s.dual_value);
      },
      py::arg("graph"), py::arg("state"), py::arg("b") = 2, py::arg("eta") = 0.5, py::arg("update") = "midpoint");
  m.def(
      "gauss_seidel_sweep",
      [](const f2m::Graph& graph, f2m::DualState& state, int b, const std::string& update) {
        const f2m::SweepStats s = f2m::gauss_seidel_sweep(
            graph, state, engine_config(b, 0.5, 1e-9, 0, "gauss-seidel", update, "local-midpoint", 0));
        return py::make_tuple(s.max_abs_delta, s.dual_value);
      },
      py::arg("graph"), py::arg("state"), py::arg("b") = 2, py::arg("update") = "midpoint");

  py::class_<f2m::PrimalSolution>(m, "PrimalSolution")
      .def_readonly("value", &f2m::PrimalSolution::value)
      .def_readonly("objective", &f2m::PrimalSolution::objective);

  m.def("classify_edges",
        [](const f2m::Graph& graph, const f2m::DualState& state, double tol) {
          const f2m::EdgeClassification c = f2m::classify_edges(graph, state, tol);
          py::array_t<uint8_t> a(static_cast<py::ssize_t>(c.label.size()));
          for (size_t e = 0; e < c.label.size(); ++e) a.mutable_data()[e] = static_cast<uint8_t>(c.label[e]);
          return a;
        },
        py::arg("graph"), py::arg("state"), py::arg("tol"));
  m.def("extract_primal", &f2m::extract_primal, py::arg("graph"), py::arg("state"), py::arg("tol"));
  m.def("solve_zero_component", &f2m::solve_zero_component, py::arg("graph"), py::arg("component_edges"),
        py::arg("residual"));
  m.def("verify_solution", [](const f2m::Graph& graph, const f2m::PrimalSolution& solution,
                              const f2m::DualState& state) {
    const f2m::VerificationReport r = f2m::verify_solution(graph, solution, state);
    return py::dict(py::arg("feasible") = r.feasible, py::arg("violated_nodes") = r.violated_nodes,
                    py::arg("duality_gap") = r.duality_gap, py::arg("value_violations") = r.value_violations);
  });
  m.def("write_solution", [](const f2m::Graph& graph, const f2m::PrimalSolution& solution,
                             const f2m::DualState& state) {
    std::ostringstream out;
    f2m::write_solution(graph, solution, f2m::verify_solution(graph, solution, state), out);
    return out.str();
  });

  m.def(
      "brute_force_f2m",
      [](const f2m::Graph& graph, int max_edges) {
        const f2m::OracleResult r = f2m::brute_force_f2m(graph, max_edges);
        return py::dict(py::arg("optimum") = r.optimum, py::arg("value") = r.solution.value,
                        py::arg("enumerated") = r.enumerated);
      },
      py::arg("graph"), py::arg("max_edges") = 20);

  m.def(
      "full_solve",
      [](const f2m::Instance& instance, int k, double eta, double eps, int max_sweeps, const std::string& mode,
         double tol, int max_restarts, std::uint64_t seed, int threads, int num_gpus) {
        f2m::RunConfig config;
        config.k = k;
        config.engine = engine_config(2, eta, eps, max_sweeps, mode, "midpoint", "local-midpoint", threads);
        config.engine.num_gpus = num_gpus;
        config.tol = tol;
        config.max_restarts = max_restarts;
        config.seed = seed;
        f2m::SolveOutcome outcome;
        {
          py::gil_scoped_release release;
          outcome = f2m::full_solve(instance, config);
        }
        return py::dict(py::arg("objective") = outcome.solution.objective,
                        py::arg("value") = outcome.solution.value,
                        py::arg("feasible") = outcome.verification.feasible,
                        py::arg("gap") = outcome.verification.duality_gap,
                        py::arg("sweeps") = outcome.convergence.sweeps, py::arg("restarts") = outcome.restarts,
                        py::arg("duals") = outcome.duals.lambda);
      },
      py::arg("instance"), py::arg("k") = 20, py::arg("eta") = 0.5, py::arg("eps") = 1e-9,
      py::arg("max_sweeps") = 20000, py::arg("mode") = "jacobi", py::arg("tol") = 0.0, py::arg("max_restarts") = 5,
      py::arg("seed") = 0, py::arg("threads") = 0, py::arg("num_gpus") = 1);

  m.def(
      "full_solve_graph",
      [](const f2m::Graph& graph, int k, double eta, double eps, int max_sweeps, const std::string& mode, double tol,
         int max_restarts, std::uint64_t seed, int threads, int num_gpus) {
        f2m::RunConfig config;
        config.k = k;
        config.engine = engine_config(2, eta, eps, max_sweeps, mode, "midpoint", "local-midpoint", threads);
        config.engine.num_gpus = num_gpus;
        config.tol = tol;
        config.max_restarts = max_restarts;
        config.seed = seed;
        f2m::SolveOutcome outcome;
        {
          py::gil_scoped_release release;
          outcome = f2m::full_solve_graph(graph, config);
        }
        return py::dict(py::arg("objective") = outcome.solution.objective,
                        py::arg("value") = outcome.solution.value,
                        py::arg("feasible") = outcome.verification.feasible,
                        py::arg("gap") = outcome.verification.duality_gap,
                        py::arg("sweeps") = outcome.convergence.sweeps, py::arg("restarts") = outcome.restarts,
                        py::arg("duals") = outcome.duals.lambda);
      },
      py::arg("graph"), py::arg("k") = 20, py::arg("eta") = 0.5, py::arg("eps") = 1e-9, py::arg("max_sweeps") = 20000,
      py::arg("mode") = "jacobi", py::arg("tol") = 0.0, py::arg("max_restarts") = 5, py::arg("seed") = 0,
      py::arg("threads") = 0, py::arg("num_gpus") = 1);

  // --- C-ABI pipeline entry points with array I/O (benchmark e2e / device-resident paths)
  m.def(
      "full_solve_arrays",
      [](py::array_t<double, py::array::c_style | py::array::forcecast> xy, bool rounded, int k, double eps,
         int max_sweeps, std::uint64_t seed, int max_restarts, double tol, py::object out_value,
         py::object out_duals) {
        const int n = static_cast<int>(xy.size() / 2);
        const int per = std::max(3, std::min(k, n - 1));
        f2m_run_config rc = run_config_c(k, 0.5, eps, max_sweeps, "jacobi", tol, max_restarts, seed, 1e-6, 1e-7);
        // results land directly in numpy buffers: m <= n * per (each node adds at most `per`
        // candidate edges), the edge-value view is trimmed to m afterwards (no copy). Callers that
        // solve repeatedly pass their own (ideally page-locked) buffers: the device->host copies
        // then run at DMA speed instead of faulting in fresh pageable pages every call.
        const py::ssize_t xcap = static_cast<py::ssize_t>(n) * per + 1;
        auto out_buffer = [](py::object o, py::ssize_t need, const char* what) {
          py::array_t<double> a;
          if (o.is_none()) return py::array_t<double>(need);
          a = py::array_t<double>::ensure(o);
          if (!a || !(a.flags() & py::array::c_style) || !a.writeable() || a.size() < need || !o.is(a))
            throw py::value_error(std::string(what) + ": expected a writable C-contiguous float64 array of at least " +
                                  std::to_string(need) + " elements");
          return a;
        };
        py::array_t<double> x = out_buffer(out_value, xcap, "out_value");
        py::array_t<double> lam = out_buffer(out_duals, std::max<py::ssize_t>(n, 1), "out_duals");
        double* px = x.mutable_data();
        double* pl = lam.mutable_data();
        f2m_solve_outcome o{};
        f2m_graph* g = nullptr;
        const double* p = xy.data();
        int st;
        {
          py::gil_scoped_release release;
          st = f2m_full_solve(n, p, rounded ? 1 : 0, &rc, px, pl, &o, &g);
        }
        f2m::check(st);
        f2m::Graph graph = f2m::Graph::adopt(g);
        py::dict d = outcome_dict(o);
        d["value"] = x[py::slice(0, static_cast<py::ssize_t>(graph.edge_count()), 1)];
        d["duals"] = lam[py::slice(0, n, 1)];
        d["graph"] = graph;
        return d;
      },
      py::arg("xy"), py::arg("rounded") = false, py::arg("k") = 10, py::arg("eps") = 1e-9,
      py::arg("max_sweeps") = 20000, py::arg("seed") = 0, py::arg("max_restarts") = 5, py::arg("tol") = 0.0,
      py::arg("out_value") = py::none(), py::arg("out_duals") = py::none());
  m.def(
      "full_solve_device",
      [](int n, std::uintptr_t d_xy, bool rounded, int k, double eps, int max_sweeps, std::uintptr_t d_x,
         std::int64_t x_capacity, std::uintptr_t d_lambda, std::uint64_t seed, int max_restarts) {
        f2m_run_config rc = run_config_c(k, 0.5, eps, max_sweeps, "jacobi", 0.0, max_restarts, seed, 1e-6, 1e-7);
        f2m_solve_outcome o{};
        int st;
        {
          py::gil_scoped_release release;
          st = f2m_full_solve_device(n, reinterpret_cast<const double*>(d_xy), rounded ? 1 : 0, &rc,
                                     reinterpret_cast<double*>(d_x), x_capacity,
                                     reinterpret_cast<double*>(d_lambda), &o, nullptr);
        }
        f2m::check(st);
        return outcome_dict(o);
      },
      py::arg("n"), py::arg("d_xy"), py::arg("rounded"), py::arg("k"), py::arg("eps"), py::arg("max_sweeps"),
      py::arg("d_x"), py::arg("x_capacity"), py::arg("d_lambda"), py::arg("seed") = 0, py::arg("max_restarts") = 5);

  // --- node-sharded multi-GPU GDP; driven by paper_2011_08170_b200/sharded.py.
  // Device pointers and CUDA streams cross as integers (torch .data_ptr() / .cuda_stream).
  struct Shard {
    f2m_shard* h = nullptr;
    f2m::Graph graph;  // keeps the graph (and its device costs) alive
    f2m_engine_config cfg{};
    ~Shard() { f2m_shard_destroy(h); }
  };
  py::class_<Shard, std::shared_ptr<Shard>>(m, "Shard")
      .def("info", [](const Shard& sh) {
        f2m_shard_info i{};
        f2m::check(f2m_shard_get_info(sh.h, &i));
        return py::dict(py::arg("n") = i.n, py::arg("rank") = i.rank, py::arg("world") = i.world,
                        py::arg("begin") = i.begin, py::arg("end") = i.end, py::arg("stride") = i.stride,
                        py::arg("slots") = i.slots);
      })
      .def("sweep",
           [](const Shard& sh, std::uintptr_t lam_full, std::uintptr_t lam_shard, std::uintptr_t max_bits,
              std::uintptr_t stream) {
             f2m::check(f2m_shard_sweep(sh.h, &sh.cfg, reinterpret_cast<const double*>(lam_full),
                                        reinterpret_cast<double*>(lam_shard),
                                        reinterpret_cast<unsigned long long*>(max_bits),
                                        reinterpret_cast<void*>(stream)));
           },
           py::arg("lam_full"), py::arg("lam_shard"), py::arg("max_bits"), py::arg("stream") = 0)
      // fused peer-memory solve (f2m_p2p_launch): all pointers are device addresses (integers)
      .def("p2p_launch",
           [](const Shard& sh, std::uintptr_t recv_pos, std::int64_t n_recv, std::uintptr_t recv_buf,
              std::uintptr_t send_pos, std::uintptr_t send_peer, std::uintptr_t send_dst, std::int64_t n_send,
              std::uintptr_t peer_recv, std::uintptr_t peer_nrecv, std::uintptr_t board, std::uintptr_t peer_board,
              std::uintptr_t lam_a, std::uintptr_t lam_b, double threshold, int max_sweeps, int ctas,
              std::uintptr_t ctl, std::uintptr_t stream) {
             f2m_p2p_plan pl{};
             pl.d_recv_pos = reinterpret_cast<const int32_t*>(recv_pos);
             pl.n_recv = n_recv;
             pl.d_recv_buf = reinterpret_cast<unsigned long long*>(recv_buf);
             pl.d_send_pos = reinterpret_cast<const int32_t*>(send_pos);
             pl.d_send_peer = reinterpret_cast<const int32_t*>(send_peer);
             pl.d_send_dst = reinterpret_cast<const int32_t*>(send_dst);
             pl.n_send = n_send;
             pl.d_peer_recv = reinterpret_cast<unsigned long long* const*>(peer_recv);
             pl.d_peer_nrecv = reinterpret_cast<const int64_t*>(peer_nrecv);
             pl.d_board = reinterpret_cast<unsigned long long*>(board);
             pl.d_peer_board = reinterpret_cast<unsigned long long* const*>(peer_board);
             f2m::check(f2m_p2p_launch(sh.h, &sh.cfg, &pl, reinterpret_cast<double*>(lam_a),
                                       reinterpret_cast<double*>(lam_b), threshold, max_sweeps, ctas,
                                       reinterpret_cast<void*>(ctl), reinterpret_cast<void*>(stream)));
           },
           py::arg("recv_pos"), py::arg("n_recv"), py::arg("recv_buf"), py::arg("send_pos"), py::arg("send_peer"),
           py::arg("send_dst"), py::arg("n_send"), py::arg("peer_recv"), py::arg("peer_nrecv"), py::arg("board"),
           py::arg("peer_board"), py::arg("lam_a"), py::arg("lam_b"), py::arg("threshold"), py::arg("max_sweeps"),
           py::arg("ctas"), py::arg("ctl"), py::arg("stream") = 0);
  m.def("generate_instance_device", [](int n, std::uint64_t seed, double box, std::uintptr_t d_xy,
                                        std::uintptr_t stream) {
    f2m::check(f2m_generate_instance_device(n, seed, box, reinterpret_cast<double*>(d_xy),
                                            reinterpret_cast<void*>(stream)));
  }, py::arg("n"), py::arg("seed"), py::arg("box"), py::arg("d_xy"), py::arg("stream") = 0);
  m.def("debug_warp_profile", []() {
    py::array_t<unsigned long long> out({160, 32, 12});
    f2m::check(f2m_debug_warp_profile(out.mutable_data(), static_cast<size_t>(out.size())));
    return out;
  });
  m.def("debug_sweep_trace", [](bool reset) {
    py::array_t<unsigned long long> out({160, 64, 4});
    f2m::check(f2m_debug_sweep_trace(out.mutable_data(), static_cast<size_t>(out.size()), reset ? 1 : 0));
    return out;
  }, py::arg("reset") = false);
  m.def("set_allpairs_mode", [](int mode) { f2m::check(f2m_set_allpairs_mode(mode)); }, py::arg("mode"));
  m.def("set_sweep_partition", [](int ctas) { f2m_set_sweep_partition(ctas); }, py::arg("ctas"));
  m.def("set_gpu_list", [](const std::vector<int>& devices) {
    f2m::check(f2m_set_gpu_list(devices.data(), static_cast<int>(devices.size())));
  }, py::arg("devices"));
  m.def("multi_gpu_info", [](const f2m::Graph& graph) {
    int w = 0, p = 0, r = 0;
    f2m::check(f2m_multi_gpu_info(graph.handle(), &w, &p, &r));
    return py::dict(py::arg("world") = w, py::arg("partition_ctas") = p, py::arg("resident") = (bool)r);
  }, py::arg("graph"));
  m.def("sweep_multi_info", [](const f2m::Graph& graph, int rank, int world) {
    int gt = 0, res = 0, b = 0, e = 0;
    std::int64_t llw = 0, cmw = 0;
    f2m::check(f2m_sweep_multi_info(graph.handle(), rank, world, &gt, &res, &llw, &cmw, &b, &e));
    return py::dict(py::arg("g_total") = gt, py::arg("resident") = (bool)res, py::arg("ll_words") = llw,
                    py::arg("cmax_words") = cmw, py::arg("begin") = b, py::arg("end") = e);
  });
  m.def("sweep_multi_ctl_bytes", []() { return f2m_sweep_multi_ctl_bytes(); });
  m.def("sweep_multi_traffic", [](const f2m::Graph& graph, int rank, int world) {
    std::int64_t ll = 0, mx = 0;
    f2m::check(f2m_sweep_multi_traffic(graph.handle(), rank, world, &ll, &mx));
    return py::dict(py::arg("remote_ll_stores") = ll, py::arg("remote_max_stores") = mx,
                    py::arg("bytes_per_sweep") = 16 * (ll + mx));
  }, py::arg("graph"), py::arg("rank"), py::arg("world"));
  m.def(
      "sweep_multi_launch",
      [](const f2m::Graph& graph, int b, double eta, const std::string& update, int rank, int world,
         std::uintptr_t ring, std::uintptr_t ll, std::uintptr_t ll_peers, std::uintptr_t cmax,
         std::uintptr_t cmax_peers, double threshold, int max_sweeps, std::uintptr_t ctl, std::uintptr_t stream) {
        f2m_engine_config c{};
        c.b = b;
        c.eta = eta;
        c.eps = 1e-9;
        c.max_sweeps = max_sweeps;
        c.update = update == "paper-difference" ? 1 : 0;
        f2m::check(f2m_sweep_multi_launch(graph.handle(), &c, rank, world, reinterpret_cast<double*>(ring),
                                          reinterpret_cast<unsigned long long*>(ll),
                                          reinterpret_cast<unsigned long long* const*>(ll_peers),
                                          reinterpret_cast<unsigned long long*>(cmax),
                                          reinterpret_cast<unsigned long long* const*>(cmax_peers), threshold,
                                          max_sweeps, reinterpret_cast<void*>(ctl), reinterpret_cast<void*>(stream)));
      },
      py::arg("graph"), py::arg("b"), py::arg("eta"), py::arg("update"), py::arg("rank"), py::arg("world"),
      py::arg("ring"), py::arg("ll"), py::arg("ll_peers"), py::arg("cmax"), py::arg("cmax_peers"),
      py::arg("threshold"), py::arg("max_sweeps"), py::arg("ctl"), py::arg("stream") = 0);
  m.def("sweep_multi_result", [](std::uintptr_t ctl) {
    int sw = 0, conv = 0, ob = 0;
    double fm = 0.0;
    f2m::check(f2m_sweep_multi_result(reinterpret_cast<const void*>(ctl), &sw, &conv, &fm, &ob));
    return py::dict(py::arg("sweeps") = sw, py::arg("converged") = (bool)conv, py::arg("final_max_abs_delta") = fm,
                    py::arg("out_buffer") = ob);
  });
  m.def("p2p_ctl_bytes", []() { return f2m_p2p_ctl_bytes(); });
  m.def("p2p_max_ctas", [](int b) {
    const int v = f2m_p2p_max_ctas(b);
    if (v < 0) f2m::check(-v);
    return v;
  }, py::arg("b") = 2);
  m.def("p2p_result", [](std::uintptr_t ctl) {
    f2m_p2p_result r{};
    f2m::check(f2m_p2p_get_result(reinterpret_cast<const void*>(ctl), &r));
    return py::dict(py::arg("sweeps") = r.sweeps, py::arg("converged") = (bool)r.converged,
                    py::arg("out_buffer") = r.out_buffer, py::arg("final_max_abs_delta") = r.final_max_abs_delta);
  });
  m.def(
      "shard_create",
      [](const f2m::Graph& graph, int rank, int world, int b, double eta, const std::string& update) {
        auto sh = std::make_shared<Shard>();
        sh->graph = graph;
        sh->cfg.b = b;
        sh->cfg.eta = eta;
        sh->cfg.eps = 1e-9;
        sh->cfg.max_sweeps = 1;
        sh->cfg.update = update == "paper-difference" ? 1 : 0;
        f2m::check(f2m_engine_config_validate(&sh->cfg));
        f2m::check(f2m_shard_create(graph.handle(), rank, world, &sh->h));
        return sh;
      },
      py::arg("graph"), py::arg("rank"), py::arg("world"), py::arg("b") = 2, py::arg("eta") = 0.5,
      py::arg("update") = "midpoint");
  m.def(
      "initial_state_positions",
      [](const f2m::Graph& graph, std::uintptr_t d_lam_pos, int b, const std::string& init, std::uintptr_t stream) {
        f2m_engine_config c{};
        c.b = b;
        c.eta = 0.5;
        c.eps = 1e-9;
        c.init = init == "zero" ? 1 : 0;
        f2m::check(f2m_initial_state_positions(graph.handle(), &c, reinterpret_cast<double*>(d_lam_pos),
                                               reinterpret_cast<void*>(stream)));
      },
      py::arg("graph"), py::arg("d_lam_pos"), py::arg("b") = 2, py::arg("init") = "local-midpoint",
      py::arg("stream") = 0);
  m.def(
      "positions_to_ids",
      [](const f2m::Graph& graph, std::uintptr_t d_pos, std::uintptr_t d_ids, std::uintptr_t stream) {
        f2m::check(f2m_positions_to_ids(graph.handle(), reinterpret_cast<const double*>(d_pos),
                                        reinterpret_cast<double*>(d_ids), reinterpret_cast<void*>(stream)));
      },
      py::arg("graph"), py::arg("d_pos"), py::arg("d_ids"), py::arg("stream") = 0);
  m.def(
      "gather_f64",
      [](std::uintptr_t src, std::uintptr_t idx, std::uintptr_t dst, std::int64_t count, std::uintptr_t stream) {
        f2m::check(f2m_gather_f64(reinterpret_cast<const double*>(src), reinterpret_cast<const int32_t*>(idx),
                                  reinterpret_cast<double*>(dst), count, reinterpret_cast<void*>(stream)));
      },
      py::arg("src"), py::arg("idx"), py::arg("dst"), py::arg("count"), py::arg("stream") = 0);
  m.def(
      "scatter_f64",
      [](std::uintptr_t src, std::uintptr_t idx, std::uintptr_t dst, std::int64_t count, std::uintptr_t stream) {
        f2m::check(f2m_scatter_f64(reinterpret_cast<const double*>(src), reinterpret_cast<const int32_t*>(idx),
                                   reinterpret_cast<double*>(dst), count, reinterpret_cast<void*>(stream)));
      },
      py::arg("src"), py::arg("idx"), py::arg("dst"), py::arg("count"), py::arg("stream") = 0);
  m.def(
      "seq_sums",
      [](std::uintptr_t v, std::int64_t k, std::int64_t seg_len, std::uintptr_t out, std::uintptr_t stream) {
        f2m::check(f2m_seq_sums(reinterpret_cast<const double*>(v), k, seg_len, reinterpret_cast<double*>(out),
                                reinterpret_cast<void*>(stream)));
      },
      py::arg("d_v"), py::arg("k"), py::arg("seg_len"), py::arg("d_out"), py::arg("stream") = 0);
  m.def(
      "ids_to_positions",
      [](const f2m::Graph& graph, std::uintptr_t d_ids, std::uintptr_t d_pos, std::uintptr_t stream) {
        f2m::check(f2m_ids_to_positions(graph.handle(), reinterpret_cast<const double*>(d_ids),
                                        reinterpret_cast<double*>(d_pos), reinterpret_cast<void*>(stream)));
      },
      py::arg("graph"), py::arg("d_ids"), py::arg("d_pos"), py::arg("stream") = 0);

  m.def("write_lp", [](const f2m::Graph& graph) {
    std::ostringstream out;
    f2m::write_lp(graph, out);
    return out.str();
  });

  // --- observability
  m.def("device_info", []() {
    f2m_device_info d{};
    f2m::check(f2m_get_device_info(&d));
    return py::dict(py::arg("device") = d.device, py::arg("sm_count") = d.sm_count,
                    py::arg("sweep_ctas") = d.sweep_ctas, py::arg("sweep_threads") = d.sweep_threads,
                    py::arg("cc") = std::to_string(d.cc_major) + "." + std::to_string(d.cc_minor),
                    py::arg("name") = std::string(d.name));
  });
  m.def("set_device", [](int dev) { f2m::check(f2m_set_device(dev)); }, py::arg("device"));
  m.def("kernel_launch_count", []() { return f2m_kernel_launch_count(); });
  m.def("last_sweep_kernel_desc", []() { return std::string(f2m_last_sweep_kernel_desc()); });
  m.def("last_sweep_kernel", []() {
    double ms = 0.0;
    int sweeps = 0;
    f2m_last_sweep_kernel_ms(&ms, &sweeps);
    return py::make_tuple(ms, sweeps);
  });
}

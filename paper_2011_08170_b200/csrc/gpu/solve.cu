// solve.cu — end-to-end pipeline (solve.cpp:51-106) over device-resident data.
//
// full_solve_graph keeps the reference's control flow — validate, then a restart loop of
// solve_duals -> extract_primal -> objective on the ORIGINAL costs -> verify_solution ->
// certify gap <= gap_tol*(1+|obj|) — but every stage runs on the device and nothing crosses
// PCIe between stages except scalars: lambda, x and the jittered costs (generated on the
// device from the counter-based SplitMix64 stream) never leave HBM until the final download.
#include <chrono>
#include <sstream>

#include <cstring>

#include "internal.cuh"

namespace f2mgpu {

static void validate_run(const f2m_run_config& rc) {
  // RunConfig::validate (solve.cpp:20-27)
  validate_engine(rc.engine);
  if (rc.k < 3) throw Error(F2M_E_ARGUMENT, "RunConfig: k must be >= 3");
  if (rc.tol < 0.0) throw Error(F2M_E_ARGUMENT, "RunConfig: tol must be >= 0");
  if (!(rc.gap_tol > 0.0)) throw Error(F2M_E_ARGUMENT, "RunConfig: gap_tol must be > 0");
  if (rc.max_restarts < 0) throw Error(F2M_E_ARGUMENT, "RunConfig: max_restarts must be >= 0");
  if (rc.perturb_scale < 0.0) throw Error(F2M_E_ARGUMENT, "RunConfig: perturb_scale must be >= 0");
}

static double effective_tol(const f2m_run_config& rc) {  // solve.cpp:16-18
  return rc.tol > 0.0 ? rc.tol : std::max(1e-7, 10.0 * rc.engine.eps);
}

static double cost_scale(const f2m_graph& g) {  // solve.cpp:33-35
  return graph_mean(g) > 0.0 ? g.mean_cost : 1.0;
}

static double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Runs the certified pipeline; on success leaves x and lambda (position order) in the
// returned device buffers.
static void full_solve_graph_device(const f2m_graph& g, const f2m_run_config& rc, DBuf<double>& d_x,
                                    DBuf<double>& d_lam, f2m_solve_outcome& out) {
  validate_run(rc);
  // validate_graph (solve.cpp:55) without a synchronisation of its own: its verdict is read after
  // the first attempt's dual solve, before any result is used
  unsigned long long* h_valid = reinterpret_cast<unsigned long long*>(pinned_scratch() + 15);
  validate_graph_async(g, h_valid);
  bool validated = false;
  const Topology& t = *g.topo;
  std::string last_failure = "no attempt made";
  double t_duals = 0.0, t_extract = 0.0;
  for (int restart = 0; restart <= rc.max_restarts; ++restart) {
    f2m_graph* jit = nullptr;
    if (restart > 0) {
      const int st = f2m_graph_jittered(&g, rc.seed, restart, rc.perturb_scale, &jit);
      if (st != F2M_OK) throw Error(st, f2m_last_error());
    }
    std::unique_ptr<f2m_graph, void (*)(f2m_graph*)> holder(jit, f2m_graph_destroy);
    const f2m_graph& attempt = jit ? *jit : g;

    auto ts = std::chrono::steady_clock::now();
    f2m_convergence_report conv{};
    DBuf<double> lam;
    // restart 0 solves g itself with b = 2: its dual objective is the certificate's g(lambda);
    // it is read back (page-locked, asynchronously) with the extraction's synchronisations
    const bool same = jit == nullptr && rc.engine.b == 2;
    double* dual_async = reinterpret_cast<double*>(pinned_scratch() + 24);
    try {
      solve_duals_device(attempt, rc.engine, nullptr, lam, conv, dual_async);
    } catch (...) {
      if (!validated) {  // a structural defect is the reference's first error
        F2M_CUDA(cudaStreamSynchronize(t.stream));
        validate_graph_check(g, *h_valid);
      }
      throw;
    }
    if (!validated) {  // solve_duals_device synchronised the stream
      validate_graph_check(g, *h_valid);
      validated = true;
    }
    t_duals += seconds_since(ts);

    ts = std::chrono::steady_clock::now();
    DBuf<double> x(std::max<int64_t>(t.m, 1), t.stream);
    try {
      extract_device(attempt, lam.get(), effective_tol(rc) * cost_scale(attempt), x.get());
    } catch (const Error& e) {
      if (e.code != F2M_E_DEGENERATE) throw;
      last_failure = e.what();
      t_extract += seconds_since(ts);
      continue;
    }
    // certify against the unperturbed costs (solve.cpp:74-83)
    const double dual = same ? 0.0 : dual_objective_device(g, lam.get(), 2);
    double objective = 0.0;
    f2m_verification ver{};
    certify_device(g, x.get(), 0.0, objective, ver);  // synchronises: the async dual is valid now
    std::memcpy(&conv.dual_value, dual_async, sizeof(double));
    ver.duality_gap = objective - (same ? conv.dual_value : dual);
    t_extract += seconds_since(ts);
    const double scale = 1.0 + std::fabs(objective);
    if (ver.feasible && ver.duality_gap <= rc.gap_tol * scale) {
      out.objective = objective;
      out.verification = ver;
      out.convergence = conv;
      out.restarts = restart;
      out.t_duals = t_duals;
      out.t_extract = t_extract;
      d_x = std::move(x);
      d_lam = std::move(lam);
      return;
    }
    std::ostringstream oss;
    oss << "uncertified attempt: feasible=" << ver.feasible << " gap=" << ver.duality_gap;
    last_failure = oss.str();
  }
  throw Error(F2M_E_SOLVE_FAILED, "restarts exhausted (" + std::to_string(rc.max_restarts) +
                                      "); last failure: " + last_failure);
}

__global__ void k_gather_pos(int n, const double* __restrict__ src, const int32_t* __restrict__ perm,
                             double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

}  // namespace f2mgpu

using namespace f2mgpu;

extern "C" int f2m_run_config_validate(const f2m_run_config* rc) {
  return guard([&] { validate_run(*rc); });
}

extern "C" int f2m_full_solve_graph(const f2m_graph* g, const f2m_run_config* rc, double* x, double* lambda,
                                    f2m_solve_outcome* out) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    const auto t0 = std::chrono::steady_clock::now();
    *out = f2m_solve_outcome{};
    DBuf<double> dx, dlam;
    full_solve_graph_device(*g, *rc, dx, dlam, *out);
    if (x && t.m > 0) F2M_CUDA(cudaMemcpyAsync(x, dx.get(), sizeof(double) * t.m, cudaMemcpyDeviceToHost, t.stream));
    if (lambda) download_lambda(*g, dlam.get(), lambda);
    F2M_CUDA(cudaStreamSynchronize(t.stream));
    out->t_total = seconds_since(t0);
  });
}

static void full_solve_impl(int n, const double* xy, bool xy_on_device, int rounded, const f2m_run_config* rc,
                            double* x, int64_t x_capacity, bool out_on_device, double* lambda,
                            f2m_solve_outcome* out, f2m_graph** graph_out) {
  validate_run(*rc);
  const int dev = current_device();
  F2M_CUDA(cudaSetDevice(dev));
  *out = f2m_solve_outcome{};
  if (graph_out) *graph_out = nullptr;
  cudaEvent_t e0, e1;
  F2M_CUDA(cudaEventCreate(&e0));
  F2M_CUDA(cudaEventCreate(&e1));
  const auto t0 = std::chrono::steady_clock::now();
  f2m_graph* g = nullptr;
  try {
    const int k = std::min(rc->k, n - 1);  // solve.cpp:103-104
    g = knn_build_device(n, xy, !xy_on_device, rounded, std::max(k, 3), dev, e0);
    out->t_knn = seconds_since(t0);
    DBuf<double> dx, dlam;
    full_solve_graph_device(*g, *rc, dx, dlam, *out);
    const Topology& t = *g->topo;
    cudaStream_t s = t.stream;
    if (out_on_device) {
      if (x) {
        if (x_capacity < t.m) throw Error(F2M_E_ARGUMENT, "full_solve_device: x capacity below edge count");
        if (t.m > 0) F2M_CUDA(cudaMemcpyAsync(x, dx.get(), sizeof(double) * t.m, cudaMemcpyDeviceToDevice, s));
      }
      if (lambda && n > 0) {
        k_gather_pos<<<grid_for(n, 256), 256, 0, s>>>(n, dlam.get(), t.perm.get(), lambda);
        launched("gather_lambda");
      }
    } else {
      if (x && t.m > 0) F2M_CUDA(cudaMemcpyAsync(x, dx.get(), sizeof(double) * t.m, cudaMemcpyDeviceToHost, s));
      if (lambda) download_lambda(*g, dlam.get(), lambda);
    }
    F2M_CUDA(cudaEventRecord(e1, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    F2M_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    out->t_total = ms * 1e-3;  // device-event time on the solve's stream
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (g) f2m_graph_destroy(g);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (graph_out) *graph_out = g;
  else f2m_graph_destroy(g);
}

extern "C" int f2m_full_solve(int n, const double* xy, int rounded, const f2m_run_config* rc, double* x,
                              double* lambda, f2m_solve_outcome* out, f2m_graph** graph_out) {
  return guard([&] { full_solve_impl(n, xy, false, rounded, rc, x, INT64_MAX, false, lambda, out, graph_out); });
}

extern "C" int f2m_full_solve_device(int n, const double* d_xy, int rounded, const f2m_run_config* rc,
                                     double* d_x, int64_t d_x_capacity, double* d_lambda,
                                     f2m_solve_outcome* out, f2m_graph** graph_out) {
  return guard([&] {
    full_solve_impl(n, d_xy, true, rounded, rc, d_x, d_x_capacity, true, d_lambda, out, graph_out);
  });
}

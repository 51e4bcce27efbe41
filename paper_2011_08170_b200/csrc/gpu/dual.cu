// dual.cu — the GDP engine on sm_100a (dual.hpp / dual.cpp).
//
//  k_gdp_sweep<B>   persistent cooperative kernel: ALL Jacobi sweeps of solve_duals
//                   (dual.cpp:227-239) in one launch. One CTA per SM owns a contiguous,
//                   slot-balanced range of SELL-32 slices (a compact Morton patch); one thread
//                   per node keeps the (B+1) smallest adjusted lengths (c - l_v) - l_u of its
//                   row (smallest_adjusted, dual.cpp:33-61) in registers, applies the midpoint
//                   update l_v + eta*delta (dual.cpp:147-160) into the other lambda buffer
//                   (double buffering == the reference's frozen snapshot) and folds |delta|
//                   into a block max. The CTA max goes to a 64-bit atomicMax on the sweep's
//                   slot, then a grid barrier; every CTA reads the global max and applies the
//                   convergence test max|delta| <= eps*mean_cost (dual.cpp:235) itself, so
//                   there is no per-sweep host round trip.
//  k_init_local_midpoint  make_initial_state (dual.cpp:194-208) is an in-order Gauss-Seidel
//                   pass from zero: node v sees the FINAL multipliers of lower-numbered
//                   neighbours. Sync-free DAG execution: warps claim nodes in id order from a
//                   global counter and spin on per-node done flags of lower neighbours.
//  k_gs_sweep       gauss_seidel_sweep (dual.cpp:175-192): one warp, nodes in id order.
//  k_dual_chunks    dual_objective (dual.cpp:87-123) in the reference's 2048/8192 chunk
//                   order: one warp per chunk, lane 0 adds in sequence -> bit-exact.
#include <chrono>

#include "internal.cuh"

namespace f2mgpu {

constexpr int kSweepThreads = 1024;

int sweep_block_threads() { return kSweepThreads; }

int sweep_grid_ctas(int dev) { return device_props(dev).multiProcessorCount; }

// ---------------------------------------------------------------- selection helpers
// Insert val into the sorted (ascending) s[0..B]; s starts at +inf. Equivalent to the
// reference's insertion into the (b+1) smallest (dual.cpp:44-58): the kept multiset is the
// b+1 smallest values of the row, whatever the visiting order.
template <int B>
__device__ __forceinline__ void topk_insert(double (&s)[B + 1], double val) {
  if (val < s[B]) {
#pragma unroll
    for (int i = B; i > 0; --i) {
      // s[i] = (val < s[i-1]) ? s[i-1] : max(val, s[i])  written branch-free
      const double hi = val < s[i - 1] ? s[i - 1] : val;
      s[i] = s[i] < hi ? s[i] : hi;
    }
    s[0] = val < s[0] ? val : s[0];
  }
}

template <int B>
__device__ __forceinline__ double delta_of(const double (&s)[B + 1], int update) {
  // delta_for (dual.cpp:63-68)
  return update ? dmul(0.5, dsub(s[B - 1], s[B])) : dmul(0.5, dadd(s[B - 1], s[B]));
}

// Butterfly merge of per-lane sorted top lists: every lane ends with the warp's B+1 smallest.
template <int B>
__device__ __forceinline__ void warp_topk_merge(double (&s)[B + 1]) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    double o[B + 1];
#pragma unroll
    for (int i = 0; i <= B; ++i) o[i] = __shfl_xor_sync(0xffffffffu, s[i], off);
#pragma unroll
    for (int i = 0; i <= B; ++i) topk_insert<B>(s, o[i]);
  }
}

// ---------------------------------------------------------------- persistent Jacobi sweep
struct SweepCtl {
  unsigned bar;
  int error;
  unsigned long long maxbits[3];
  int sweeps;
  int converged;
  double final_max;
};

struct SweepArgs {
  int n;
  const int64_t* __restrict__ sptr;
  const int32_t* __restrict__ swidth;
  const int32_t* __restrict__ scol;
  const double* __restrict__ scost;
  const int32_t* __restrict__ cta_lo;
  double* lam0;
  double* lam1;
  double eta;
  int update;
  double threshold;
  int max_sweeps;
  double* record;  // per-sweep global max |delta| (nullable)
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target, int* err) {
  // thread 0 of each CTA, between two __syncthreads (cooperative-groups grid.sync pattern)
  __threadfence();
  atomicAdd(bar, 1u);
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_u32(bar) < target) {
    if (globaltimer_ns() - t0 > 20ull * 1000000000ull) {  // 20 s watchdog: never hang the GPU
      atomicExch(err, 1);
      break;
    }
  }
  __threadfence();
}

template <int B>
__global__ void __launch_bounds__(kSweepThreads, 1) k_gdp_sweep(SweepArgs a, SweepCtl* ctl) {
  __shared__ double red[kSweepThreads / 32];
  __shared__ double s_gmax;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int s_lo = a.cta_lo[blockIdx.x];
  const int s_hi = a.cta_lo[blockIdx.x + 1];

  int sweep = 0;
  double gmax = INFINITY;
  bool converged = false;
  for (; sweep < a.max_sweeps; ++sweep) {
    const double* lin = (sweep & 1) ? a.lam1 : a.lam0;
    double* lout = (sweep & 1) ? a.lam0 : a.lam1;
    double mx = 0.0;
    for (int sl = s_lo + warp; sl < s_hi; sl += nwarps) {
      const int p = sl * 32 + lane;
      if (p >= a.n) continue;
      const int64_t base = a.sptr[sl] + lane;
      const int w = a.swidth[sl];
      const double lv = lin[p];
      double s[B + 1];
#pragma unroll
      for (int i = 0; i <= B; ++i) s[i] = CUDART_INF;
      int j = 0;
      for (; j + 4 <= w; j += 4) {  // 4 independent gathers in flight per thread
        int q[4];
        double c[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          q[u] = a.scol[base + (int64_t)(j + u) * 32];
          c[u] = a.scost[base + (int64_t)(j + u) * 32];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) l[u] = lin[q[u]];
#pragma unroll
        for (int u = 0; u < 4; ++u) topk_insert<B>(s, dsub(dsub(c[u], lv), l[u]));
      }
      for (; j < w; ++j) {
        const int q = a.scol[base + (int64_t)j * 32];
        const double c = a.scost[base + (int64_t)j * 32];
        topk_insert<B>(s, dsub(dsub(c, lv), lin[q]));
      }
      const double d = delta_of<B>(s, a.update);
      lout[p] = dadd(lv, dmul(a.eta, d));
      const double ad = fabs(d);
      mx = mx < ad ? ad : mx;  // std::max(local_max, |d|) (dual.cpp:149)
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, mx, off);
      mx = mx < o ? o : mx;
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double bm = 0.0;
      for (int w = 0; w < nwarps; ++w) bm = bm < red[w] ? red[w] : bm;
      if (blockIdx.x == 0) ctl->maxbits[(sweep + 1) % 3] = 0ull;  // next sweep's slot
      atomicMax(&ctl->maxbits[sweep % 3], (unsigned long long)__double_as_longlong(bm));
      grid_barrier(&ctl->bar, (unsigned)(sweep + 1) * gridDim.x, &ctl->error);
      const unsigned long long bits =
          atomicAdd(&ctl->maxbits[sweep % 3], 0ull);  // coherent read after the barrier
      s_gmax = __longlong_as_double((long long)bits);
      if (blockIdx.x == 0 && a.record) a.record[sweep] = s_gmax;
    }
    __syncthreads();
    gmax = s_gmax;
    if (ctl->error) break;
    if (gmax <= a.threshold) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->sweeps = sweep;
    ctl->converged = converged ? 1 : 0;
    ctl->final_max = gmax;
  }
}

static double g_last_sweep_ms = 0.0;
static int g_last_sweep_count = 0;

template <int B>
static void launch_sweep(const SweepArgs& a, SweepCtl* ctl, int ctas, cudaStream_t s) {
  void* args[] = {(void*)&a, (void*)&ctl};
  F2M_CUDA(cudaLaunchCooperativeKernel((const void*)k_gdp_sweep<B>, dim3(ctas), dim3(kSweepThreads),
                                       args, 0, s));
}

SweepResult run_jacobi(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam0,
                       double* d_lam1, int max_sweeps, double threshold, double* d_record) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  SweepResult r;
  if (max_sweeps <= 0) return r;
  DBuf<SweepCtl> ctl(1, s);
  F2M_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(SweepCtl), s));
  SweepArgs a;
  a.n = t.n;
  a.sptr = t.sptr.get();
  a.swidth = t.swidth.get();
  a.scol = t.scol.get();
  a.scost = g.scost.get();
  a.cta_lo = t.cta_lo.get();
  a.lam0 = d_lam0;
  a.lam1 = d_lam1;
  a.eta = cfg.eta;
  a.update = cfg.update;
  a.threshold = threshold;
  a.max_sweeps = max_sweeps;
  a.record = d_record;
  cudaEvent_t e0, e1;
  F2M_CUDA(cudaEventCreate(&e0));
  F2M_CUDA(cudaEventCreate(&e1));
  F2M_CUDA(cudaEventRecord(e0, s));
  switch (cfg.b) {
    case 1: launch_sweep<1>(a, ctl.get(), t.sweep_ctas, s); break;
    case 2: launch_sweep<2>(a, ctl.get(), t.sweep_ctas, s); break;
    case 3: launch_sweep<3>(a, ctl.get(), t.sweep_ctas, s); break;
    case 4: launch_sweep<4>(a, ctl.get(), t.sweep_ctas, s); break;
    case 5: launch_sweep<5>(a, ctl.get(), t.sweep_ctas, s); break;
    case 6: launch_sweep<6>(a, ctl.get(), t.sweep_ctas, s); break;
    case 7: launch_sweep<7>(a, ctl.get(), t.sweep_ctas, s); break;
    default: launch_sweep<8>(a, ctl.get(), t.sweep_ctas, s); break;
  }
  launched("gdp_sweep");
  F2M_CUDA(cudaEventRecord(e1, s));
  SweepCtl h;
  F2M_CUDA(cudaMemcpyAsync(&h, ctl.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_last_sweep_ms = ms;
  g_last_sweep_count = h.sweeps;
  if (h.error) throw Error(F2M_E_TIMEOUT, "gdp sweep kernel: grid barrier watchdog fired");
  r.sweeps = h.sweeps;
  r.converged = h.converged;
  r.final_max_abs_delta = h.final_max;
  r.out_buffer = (h.sweeps & 1) ? 1 : 0;
  return r;
}

// ---------------------------------------------------------------- init (make_initial_state)
template <int B>
__global__ void __launch_bounds__(256) k_init_local_midpoint(
    int n, const int32_t* __restrict__ perm, const int32_t* __restrict__ iperm,
    const int32_t* __restrict__ deg, const int64_t* __restrict__ sptr,
    const int32_t* __restrict__ scol, const double* __restrict__ scost, double* lam, int* done,
    int* counter, int* err) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int v = 0;
    if (lane == 0) v = atomicAdd(counter, 1);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v >= n) break;
    const int p = perm[v];
    const int d = deg[p];
    const int64_t base = sptr[p >> 5] + (p & 31);
    double s[B + 1];
#pragma unroll
    for (int i = 0; i <= B; ++i) s[i] = CUDART_INF;
    for (int j = lane; j < d; j += 32) {
      const int q = scol[base + (int64_t)j * 32];
      const double c = scost[base + (int64_t)j * 32];
      double other = 0.0;  // lambda of a higher-numbered (or the same) node is still 0
      if (iperm[q] < v) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire(done + q) == 0) {
          if (globaltimer_ns() - t0 > 20ull * 1000000000ull) { atomicExch(err, 1); break; }
        }
        other = __ldcg(lam + q);
      }
      // ge.cost - lv - other with lv = lambda[v] = 0 (dual.cpp:43)
      topk_insert<B>(s, dsub(dsub(c, 0.0), other));
    }
    warp_topk_merge<B>(s);
    if (lane == 0) {
      lam[p] = d > B ? dmul(0.5, dadd(s[B - 1], s[B])) : 0.0;
      __threadfence();
      st_release(done + p, 1);
    }
  }
}

template <int B>
static void launch_init(const f2m_graph& g, double* d_lam, int* done, int* counter, int* err) {
  const Topology& t = *g.topo;
  const int blocks = std::max(1, std::min<int>(grid_for((int64_t)t.n * 32, 256),
                                               device_props(t.dev).multiProcessorCount * 8));
  k_init_local_midpoint<B><<<blocks, 256, 0, t.stream>>>(t.n, t.perm.get(), t.iperm.get(), t.deg.get(),
                                                        t.sptr.get(), t.scol.get(), g.scost.get(), d_lam,
                                                        done, counter, err);
  launched("init_local_midpoint");
}

void initial_state_device(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam_pos) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  if (t.n == 0) return;
  F2M_CUDA(cudaMemsetAsync(d_lam_pos, 0, sizeof(double) * t.n, s));
  if (cfg.init != 0) return;  // kZero
  DBuf<int> flags(t.n + 2, s);
  F2M_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int) * (t.n + 2), s));
  int* done = flags.get();
  int* counter = flags.get() + t.n;
  int* err = flags.get() + t.n + 1;
  switch (cfg.b) {
    case 1: launch_init<1>(g, d_lam_pos, done, counter, err); break;
    case 2: launch_init<2>(g, d_lam_pos, done, counter, err); break;
    case 3: launch_init<3>(g, d_lam_pos, done, counter, err); break;
    case 4: launch_init<4>(g, d_lam_pos, done, counter, err); break;
    case 5: launch_init<5>(g, d_lam_pos, done, counter, err); break;
    case 6: launch_init<6>(g, d_lam_pos, done, counter, err); break;
    case 7: launch_init<7>(g, d_lam_pos, done, counter, err); break;
    default: launch_init<8>(g, d_lam_pos, done, counter, err); break;
  }
  int herr = 0;
  F2M_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  if (herr) throw Error(F2M_E_TIMEOUT, "initial-state kernel: dependency wait watchdog fired");
}

// ---------------------------------------------------------------- Gauss-Seidel + node delta
template <int B>
__device__ __forceinline__ double row_delta_warp(int p, int d, const int64_t* __restrict__ sptr,
                                                 const int32_t* __restrict__ scol,
                                                 const double* __restrict__ scost,
                                                 const double* lam, int update) {
  const int lane = threadIdx.x & 31;
  const int64_t base = sptr[p >> 5] + (p & 31);
  const double lv = __ldcg(lam + p);
  double s[B + 1];
#pragma unroll
  for (int i = 0; i <= B; ++i) s[i] = CUDART_INF;
  for (int j = lane; j < d; j += 32) {
    const int q = scol[base + (int64_t)j * 32];
    const double c = scost[base + (int64_t)j * 32];
    topk_insert<B>(s, dsub(dsub(c, lv), __ldcg(lam + q)));
  }
  warp_topk_merge<B>(s);
  return delta_of<B>(s, update);
}

template <int B>
__global__ void k_gs_sweep(int n, const int32_t* __restrict__ perm, const int32_t* __restrict__ deg,
                           const int64_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                           const double* __restrict__ scost, double* lam, int update,
                           double* out_max) {
  double mx = 0.0;
  for (int v = 0; v < n; ++v) {
    const int p = perm[v];
    const double d = row_delta_warp<B>(p, deg[p], sptr, scol, scost, lam, update);
    __syncwarp();
    if (threadIdx.x == 0) {
      lam[p] = dadd(__ldcg(lam + p), d);  // lambda[v] += d (dual.cpp:187), full step
      __threadfence();
      const double ad = fabs(d);
      mx = mx < ad ? ad : mx;
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) *out_max = mx;
}

template <int B>
__global__ void k_node_delta(int p, int d, const int64_t* __restrict__ sptr,
                             const int32_t* __restrict__ scol, const double* __restrict__ scost,
                             const double* lam, double* out) {
  const double r = row_delta_warp<B>(p, d, sptr, scol, scost, lam, 0);
  if (threadIdx.x == 0) *out = r;
}

// ---------------------------------------------------------------- dual objective
__global__ void __launch_bounds__(256) k_dual_chunks(int n, int64_t m, int nchunks_node,
                                                     int nchunks_edge, const int32_t* __restrict__ perm,
                                                     const int32_t* __restrict__ eu,
                                                     const int32_t* __restrict__ ev,
                                                     const double* __restrict__ cost,
                                                     const double* __restrict__ lam,
                                                     double* __restrict__ parts) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nchunks_node + nchunks_edge) return;
  double acc = 0.0;
  if (w < nchunks_node) {
    // node chunk: acc += lambda[v] for v in chunk, in order (dual.cpp:96-100)
    const int64_t b = (int64_t)w * kNodeChunk, e = min64(n, b + kNodeChunk);
    for (int64_t base = b; base < e; base += 32) {
      const int64_t v = base + lane;
      const double val = v < e ? lam[perm[v]] : 0.0;
      const int cnt = (int)min64(32, e - base);
      for (int i = 0; i < cnt; ++i) {
        const double x = __shfl_sync(0xffffffffu, val, i);
        if (lane == 0) acc = dadd(acc, x);
      }
    }
  } else {
    // edge chunk: if (v_e < 0) acc += v_e, v_e = (c - l_u) - l_v (dual.cpp:101-109)
    const int c = w - nchunks_node;
    const int64_t b = (int64_t)c * kEdgeChunk, e = min64(m, b + kEdgeChunk);
    for (int64_t base = b; base < e; base += 32) {
      const int64_t ed = base + lane;
      double val = 0.0;
      if (ed < e) val = dsub(dsub(cost[ed], lam[perm[eu[ed]]]), lam[perm[ev[ed]]]);
      unsigned neg = __ballot_sync(0xffffffffu, ed < e && val < 0.0);
      while (neg) {
        const int i = __ffs(neg) - 1;
        neg &= neg - 1;
        const double x = __shfl_sync(0xffffffffu, val, i);
        if (lane == 0) acc = dadd(acc, x);
      }
    }
  }
  if (lane == 0) parts[w] = acc;
}

__global__ void k_dual_combine(int nchunks_node, int nchunks_edge, int b, const double* __restrict__ parts,
                               double* __restrict__ out) {
  // combine_partials (parallel.cpp:102-106) in chunk order; b*node + edge (dual.cpp:122)
  double ns = 0.0, es = 0.0;
  for (int i = 0; i < nchunks_node; ++i) ns = dadd(ns, parts[i]);
  for (int i = 0; i < nchunks_edge; ++i) es = dadd(es, parts[nchunks_node + i]);
  *out = dadd(dmul((double)b, ns), es);
}

double dual_objective_device(const f2m_graph& g, const double* d_lam_pos, int b) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int nn = (int)((t.n + kNodeChunk - 1) / kNodeChunk);
  const int ne = (int)((t.m + kEdgeChunk - 1) / kEdgeChunk);
  DBuf<double> parts(nn + ne + 1, s);
  if (nn + ne > 0) {
    k_dual_chunks<<<grid_for((int64_t)(nn + ne) * 32, 256), 256, 0, s>>>(
        t.n, t.m, nn, ne, t.perm.get(), t.eu.get(), t.ev.get(), g.cost.get(), d_lam_pos, parts.get());
    launched("dual_chunks");
  }
  k_dual_combine<<<1, 1, 0, s>>>(nn, ne, b, parts.get(), parts.get() + nn + ne);
  launched("dual_combine");
  double h = 0.0;
  F2M_CUDA(cudaMemcpyAsync(&h, parts.get() + nn + ne, sizeof(double), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  return h;
}

// ---------------------------------------------------------------- validation + drivers
void validate_engine(const f2m_engine_config& c) {
  // EngineConfig::validate (dual.cpp:13-18) + the kMaxB bound (dual.cpp:70, 78)
  if (c.b < 1) throw Error(F2M_E_ARGUMENT, "EngineConfig: b must be >= 1");
  if (c.b > kMaxB) throw Error(F2M_E_ARGUMENT, "EngineConfig: b must be <= 8");
  if (!(c.eta > 0.0) || c.eta > 1.0) throw Error(F2M_E_ARGUMENT, "EngineConfig: eta must be in (0, 1]");
  if (!(c.eps > 0.0)) throw Error(F2M_E_ARGUMENT, "EngineConfig: eps must be > 0");
  if (c.max_sweeps < 0) throw Error(F2M_E_ARGUMENT, "EngineConfig: max_sweeps must be >= 0");
}

static void check_degree(const f2m_graph& g, int b) {
  const Topology& t = *g.topo;
  if (t.n > 0 && t.min_deg <= b) {
    throw Error(F2M_E_DEGREE, "node has degree " + std::to_string(t.min_deg) + " <= b = " + std::to_string(b));
  }
}

template <int B>
static void launch_gs(const f2m_graph& g, double* lam, int update, double* out_max) {
  const Topology& t = *g.topo;
  k_gs_sweep<B><<<1, 32, 0, t.stream>>>(t.n, t.perm.get(), t.deg.get(), t.sptr.get(), t.scol.get(),
                                        g.scost.get(), lam, update, out_max);
  launched("gs_sweep");
}

static double gs_sweep_device(const f2m_graph& g, const f2m_engine_config& cfg, double* lam) {
  const Topology& t = *g.topo;
  DBuf<double> mx(1, t.stream);
  switch (cfg.b) {
    case 1: launch_gs<1>(g, lam, cfg.update, mx.get()); break;
    case 2: launch_gs<2>(g, lam, cfg.update, mx.get()); break;
    case 3: launch_gs<3>(g, lam, cfg.update, mx.get()); break;
    case 4: launch_gs<4>(g, lam, cfg.update, mx.get()); break;
    case 5: launch_gs<5>(g, lam, cfg.update, mx.get()); break;
    case 6: launch_gs<6>(g, lam, cfg.update, mx.get()); break;
    case 7: launch_gs<7>(g, lam, cfg.update, mx.get()); break;
    default: launch_gs<8>(g, lam, cfg.update, mx.get()); break;
  }
  double h = 0.0;
  F2M_CUDA(cudaMemcpyAsync(&h, mx.get(), sizeof(double), cudaMemcpyDeviceToHost, t.stream));
  F2M_CUDA(cudaStreamSynchronize(t.stream));
  return h;
}

void solve_duals_device(const f2m_graph& g, const f2m_engine_config& cfg, const double* d_init,
                        DBuf<double>& d_lam_out, f2m_convergence_report& rep) {
  validate_engine(cfg);
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const auto t0 = std::chrono::steady_clock::now();
  DBuf<double> l0(std::max(t.n, 1), s), l1(std::max(t.n, 1), s);
  if (d_init) {
    if (t.n > 0)
      F2M_CUDA(cudaMemcpyAsync(l0.get(), d_init, sizeof(double) * t.n, cudaMemcpyDeviceToDevice, s));
  } else {
    initial_state_device(g, cfg, l0.get());
  }
  const double threshold = cfg.eps * g.mean_cost;  // dual.cpp:221
  rep.converged = 0;
  rep.sweeps = 0;
  rep.final_max_abs_delta = INFINITY;
  DBuf<double>* result = &l0;
  if (cfg.max_sweeps > 0) {
    check_degree(g, cfg.b);
    if (cfg.mode == 0) {
      SweepResult r = run_jacobi(g, cfg, l0.get(), l1.get(), cfg.max_sweeps, threshold, nullptr);
      rep.sweeps = r.sweeps;
      rep.converged = r.converged;
      rep.final_max_abs_delta = r.final_max_abs_delta;
      result = r.out_buffer ? &l1 : &l0;
    } else {
      for (int sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        const double mx = gs_sweep_device(g, cfg, l0.get());
        rep.sweeps = sweep;
        rep.final_max_abs_delta = mx;
        if (mx <= threshold) {
          rep.converged = 1;
          break;
        }
      }
    }
  }
  rep.dual_value = dual_objective_device(g, result->get(), cfg.b);
  d_lam_out = std::move(*result);
  rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace f2mgpu

using namespace f2mgpu;

// ====================================================================== C ABI

extern "C" int f2m_engine_config_validate(const f2m_engine_config* cfg) {
  return guard([&] { validate_engine(*cfg); });
}

extern "C" int f2m_initial_state(const f2m_graph* g, const f2m_engine_config* cfg, double* lambda_out) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (cfg->b < 1 || cfg->b > kMaxB) throw Error(F2M_E_ARGUMENT, "make_initial_state: b out of range");
    DBuf<double> lam(std::max(t.n, 1), t.stream);
    initial_state_device(*g, *cfg, lam.get());
    download_lambda(*g, lam.get(), lambda_out);
  });
}

extern "C" int f2m_jacobi_sweeps(const f2m_graph* g, const f2m_engine_config* cfg, double* lambda_inout,
                                 int count, double* max_abs_delta, double* dual_value) {
  return guard([&] {
    validate_engine(*cfg);
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (count < 0) throw Error(F2M_E_ARGUMENT, "jacobi_sweeps: negative count");
    cudaStream_t s = t.stream;
    DBuf<double> l0(std::max(t.n, 1), s), l1(std::max(t.n, 1), s), rec(std::max(count, 1), s);
    upload_lambda(*g, lambda_inout, l0.get());
    double* out = l0.get();
    if (count > 0) {
      check_degree(*g, cfg->b);
      // threshold -1: never converges, runs exactly `count` sweeps
      SweepResult r = run_jacobi(*g, *cfg, l0.get(), l1.get(), count, -1.0, rec.get());
      out = r.out_buffer ? l1.get() : l0.get();
      if (max_abs_delta)
        F2M_CUDA(cudaMemcpyAsync(max_abs_delta, rec.get(), sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    }
    if (dual_value) *dual_value = dual_objective_device(*g, out, cfg->b);
    download_lambda(*g, out, lambda_inout);
  });
}

extern "C" int f2m_gauss_seidel_sweeps(const f2m_graph* g, const f2m_engine_config* cfg,
                                       double* lambda_inout, int count, double* max_abs_delta,
                                       double* dual_value) {
  return guard([&] {
    validate_engine(*cfg);
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    DBuf<double> l0(std::max(t.n, 1), t.stream);
    upload_lambda(*g, lambda_inout, l0.get());
    if (count > 0) check_degree(*g, cfg->b);
    for (int i = 0; i < count; ++i) {
      const double mx = gs_sweep_device(*g, *cfg, l0.get());
      if (max_abs_delta) max_abs_delta[i] = mx;
    }
    if (dual_value) *dual_value = dual_objective_device(*g, l0.get(), cfg->b);
    download_lambda(*g, l0.get(), lambda_inout);
  });
}

extern "C" int f2m_dual_objective(const f2m_graph* g, const double* lambda, int b, double* out) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    DBuf<double> l0(std::max(t.n, 1), t.stream);
    upload_lambda(*g, lambda, l0.get());
    *out = dual_objective_device(*g, l0.get(), b);
  });
}

extern "C" int f2m_node_update_delta(const f2m_graph* g, const double* lambda, int v, int b, double* out) {
  return guard([&] {
    const Topology& t = *g->topo;
    if (v < 0 || v >= t.n) throw Error(F2M_E_INDEX, "node id out of range: " + std::to_string(v));
    if (b < 1 || b > kMaxB) throw Error(F2M_E_ARGUMENT, "node_update_delta: b out of range");
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    int p = 0, d = 0;
    F2M_CUDA(cudaMemcpyAsync(&p, t.perm.get() + v, sizeof(int), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    F2M_CUDA(cudaMemcpyAsync(&d, t.deg.get() + p, sizeof(int), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    if (d <= b)
      throw Error(F2M_E_DEGREE, "node " + std::to_string(v) + " has degree " + std::to_string(d) +
                                    " <= b = " + std::to_string(b));
    DBuf<double> l0(std::max(t.n, 1), s), res(1, s);
    upload_lambda(*g, lambda, l0.get());
    switch (b) {
#define F2M_ND(BB) case BB: k_node_delta<BB><<<1, 32, 0, s>>>(p, d, t.sptr.get(), t.scol.get(), g->scost.get(), l0.get(), res.get()); break;
      F2M_ND(1) F2M_ND(2) F2M_ND(3) F2M_ND(4) F2M_ND(5) F2M_ND(6) F2M_ND(7) F2M_ND(8)
#undef F2M_ND
    }
    launched("node_delta");
    F2M_CUDA(cudaMemcpyAsync(out, res.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int f2m_solve_duals(const f2m_graph* g, const f2m_engine_config* cfg, const double* lambda_init,
                               double* lambda_out, f2m_convergence_report* report) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    validate_engine(*cfg);
    const auto t0 = std::chrono::steady_clock::now();
    DBuf<double> init, out;
    if (lambda_init) {
      init.alloc(std::max(t.n, 1), t.stream);
      upload_lambda(*g, lambda_init, init.get());
    }
    solve_duals_device(*g, *cfg, lambda_init ? init.get() : nullptr, out, *report);
    download_lambda(*g, out.get(), lambda_out);
    report->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

extern "C" int f2m_last_sweep_kernel_ms(double* ms, int* sweeps) {
  if (ms) *ms = g_last_sweep_ms;
  if (sweeps) *sweeps = g_last_sweep_count;
  return F2M_OK;
}

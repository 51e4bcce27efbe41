// internal.cuh — shared internals of libf2m_gpu.so (sm_100a).
//
// Device data layout:
//   edge list   eu/ev int32[m], cost fp64[m]      reference edge order: (u, v) sorted, u < v
//   perm/iperm  int32[n]                          node id <-> device position (Morton order of
//                                                 the k-NN grid cells; identity for from_edges)
//   SELL-32     sptr int64[S+1], swidth int32[S]  slice s = positions 32s..32s+31; slot j of
//               scol int32[], scost fp64[]        position p lives at sptr[s] + 32*j + (p&31):
//               seid int32[]                      one coalesced 128 B col / 256 B cost line per
//                                                 warp per j. Padding: col = p, cost = +inf,
//                                                 eid = -1 (never selected: inf < s_b is false).
//   lambda      fp64[n] in position order, double buffered by the sweep kernel.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "f2m_gpu.h"

namespace f2mgpu {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

void set_last_error(const std::string& msg);

#define F2M_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      throw ::f2mgpu::Error(e_ == cudaErrorMemoryAllocation ? F2M_E_NOMEM : F2M_E_CUDA,   \
                            std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                                __FILE__ + ":" + std::to_string(__LINE__));               \
    }                                                                                     \
  } while (0)

// Wraps a C-ABI body: converts exceptions to status codes + thread-local message.
template <class F>
int guard(F&& f) {
  try {
    f();
    return F2M_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failure");
    return F2M_E_NOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return F2M_E_CUDA;
  }
}

// Kernel launch accounting (f2m_kernel_launch_count) + launch error check.
extern std::atomic<uint64_t> g_launches;
inline void launched(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    throw Error(F2M_E_CUDA, std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
  }
}

int current_device();
const cudaDeviceProp& device_props(int dev);

// ---------------------------------------------------------------- device buffers
// Stream-ordered allocation (cudaMallocAsync) so scratch reuse is cheap.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) F2M_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

#ifndef F2M_ROW_SKIP
#define F2M_ROW_SKIP 1  // per-row tail budgets of the resident head-first scans (dual.cu row_budget)
#endif
#ifndef F2M_LAM_RING8
#define F2M_LAM_RING8 1
#endif

// ---------------------------------------------------------------- graph structures
struct Topology {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int n = 0;
  int64_t m = 0;
  DBuf<int32_t> eu, ev;        // [m] sorted (u, v), u <= v (self-loops kept)
  DBuf<int32_t> perm, iperm;   // [n]
  DBuf<int32_t> perm0, iperm0; // [n] the spatial order before the CTA-local reorder (re-partitioning)
  DBuf<int32_t> deg;           // [n] by position
  int64_t nslices = 0;
  int64_t sell_slots = 0;
  DBuf<int64_t> sptr;          // [nslices+1]
  DBuf<int32_t> swidth;        // [nslices]
  DBuf<int32_t> scol;          // [sell_slots]
  DBuf<int32_t> seid;          // [sell_slots]
  int min_deg = 0, max_deg = 0;
  // persistent-sweep partition: CTA c owns slices [cta_lo[c], cta_lo[c+1])
  int sweep_ctas = 0;
  DBuf<int32_t> cta_lo;        // [sweep_ctas+1]
  DBuf<int32_t> cta_int_hi;    // [sweep_ctas]: slices [cta_lo[c], cta_int_hi[c]) hold only interior
                               // nodes (no neighbour outside the CTA); boundary nodes follow
  // v2 sweep (neighbour-flag synchronised): per-CTA local index space. Local index li of
  // CTA c: li < own_c -> position p0_c + li; else halo[halo_off[c] + li - own_c]. Every slot
  // also carries its neighbour's local index (slidx, uint16), so a sweep gathers each distinct
  // lambda once into shared memory and all slot reads hit shared memory.
  bool v2 = false;             // local index space built (max local count <= 65535)
  bool resident = false;       // per-CTA slot data (cost + slidx) fits in shared memory
  DBuf<int32_t> halo_off;      // [ctas+1]
  DBuf<int32_t> halo;          // positions (sorted per CTA)
  DBuf<uint16_t> slidx;        // [sell_slots]
  // LL halo exchange: CTA c's boundary nodes are positions [p0_c + nint_c, p1_c);
  // boundary node p publishes its multiplier at LL index boff[c] + (p - p0_c - nint_c).
  DBuf<int32_t> cta_nint;      // [ctas] interior node count
  DBuf<int32_t> boff;          // [ctas+1] exclusive prefix of boundary counts
  DBuf<int32_t> halo_pub;      // [halo entries] LL index of each halo node
  int nboundary = 0;           // total boundary nodes (LL entries per ring slot)
  // v5 split boundary rows: the sweep kernel keeps each row's slots in the order (own-CTA
  // neighbours, then halo neighbours), so the part of a boundary row that does not depend on
  // other CTAs is scanned while the halo is still in flight.
  DBuf<int32_t> sdest;         // [sell_slots] slot index in the halo-last order
  DBuf<uint8_t> row_nhalo;     // [n] halo slots in the row of each position
  int max_local = 0;           // max over CTAs of own + halo
  int max_halo = 0;            // max over CTAs of halo entries
  int64_t max_cta_slots = 0;   // max over CTAs of padded slots
  int64_t max_cta_lid4 = 0;    // max over CTAs of packed local-index entries (ushort4, widths padded to 4)
  size_t smem_bytes = 0;       // dynamic shared memory of the v2 sweep kernel
  int lam_ring = 2;            // resident: shared-memory multiplier regions (8 when they fit, see dual.cu)
  int row_skip = 0;            // resident: per-row tail budgets in shared memory (dual.cu row_budget)
  int partition_override = 0;  // > 0: partition CTA count for finalize_topology (multi-GPU replicas)
  ~Topology();
};

struct MultiPlan;  // multi.cu: per-graph replicas + rings of the single-process multi-GPU solve

}  // namespace f2mgpu
struct f2m_graph;
namespace f2mgpu {
void validate_graph_async(const f2m_graph& g, unsigned long long* h_first);
void validate_graph_check(const f2m_graph& g, unsigned long long h);

}  // namespace f2mgpu

struct f2m_graph {
  std::shared_ptr<f2mgpu::Topology> topo;
  f2mgpu::DBuf<double> cost;   // [m] reference edge order
  f2mgpu::DBuf<double> scost;  // [sell_slots] per SELL slot (+inf on padding)
  // mean_cost (graph.cpp:47-49, a SEQUENTIAL fp64 sum in edge order) is computed lazily: the
  // GDP sweep kernel computes it itself, off the critical path, on the first solve (its master
  // CTA decides early verdicts from a parallel estimate with a rigorous error bound).
  mutable double mean_cost = 0.0;
  mutable bool mean_known = false;
  f2mgpu::DBuf<double> approx_sum;  // [1] parallel sum of the costs (device)
  // Complete graph whose costs are the points' distances (build_knn_graph with k >= n-1,
  // graph.cpp:175): the sweeps can recompute every cost on the fly from the points instead of
  // streaming the n(n-1)/2-edge CSR (all-pairs mode). Points in position order.
  f2mgpu::DBuf<double2> pts_pos;
  mutable f2mgpu::DBuf<double> dense;  // all-pairs DENSE form: n x n distances, built on first use
  int rounded = 0;
  bool allpairs = false;
  // num_gpus > 1 solves: the graph replicated onto every GPU (partitioned into world x Gp CTAs)
  // and the rings of the multi-rank sweep kernel, built on first use and kept with the graph
  mutable std::shared_ptr<f2mgpu::MultiPlan> multi;
};

namespace f2mgpu {

constexpr int kMaxB = 8;          // dual.cpp:70
constexpr int kNodeChunk = 2048;  // parallel.hpp:15
constexpr int kEdgeChunk = 8192;  // parallel.hpp:16
constexpr int kMaxComponentEdges = 20;  // primal.cpp:17

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// Small page-locked host scratch (per thread, allocated once): device->host reads of several
// scalars are queued asynchronously into it and collected with ONE stream synchronisation
// (a D2H copy into pageable memory is itself synchronous). 64 int64 slots: 0-15 topology
// build, 20 init watchdog, 24 dual objective, 26-28 certification, 32-47 sweep control
// block, 48 deferred mean, 50-57 k-NN grid parameters, 58 k-NN edge count.
int64_t* pinned_scratch();
extern int g_sweep_partition;  // f2m_set_sweep_partition

// number of bits needed to represent v >= 0 (0 -> 0)
inline int bit_width(int64_t v) {
  int b = 0;
  while (v > 0) {
    ++b;
    v >>= 1;
  }
  return b;
}

inline unsigned grid_for(int64_t items, int block) {
  int64_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (1 << 30)) g = 1 << 30;
  return static_cast<unsigned>(g);
}

// Shared building blocks (core.cu)
std::shared_ptr<Topology> make_topology(int n, int dev);  // owns a fresh non-blocking stream
// Sorts + normalizes device edges in place into eu/ev/cost (stable by (u,v)).
void sort_edges(Topology& t, DBuf<int32_t>& eu, DBuf<int32_t>& ev, DBuf<double>& cost);
// Builds degrees, SELL-32 layout and the persistent-sweep partition for the given perm.
void finalize_topology(Topology& t);
// Identity permutation.
void identity_perm(Topology& t);
// cost -> scost, mean_cost (bit-exact sequential sum on the device).
void attach_costs(f2m_graph& g);
double sequential_mean(const double* d_cost, int64_t m, cudaStream_t s);
// out[j] = the left-to-right fp64 sum (from +0.0, __dadd_rn) of v[j*seg_len, min((j+1)*seg_len, k)),
// bit-exact with a sequential loop, evaluated in parallel (seqsum.cu). seg_len <= 0: one segment.
void seq_sums_device(const double* v, int64_t k, int64_t seg_len, double* out, cudaStream_t s);
// The graph's mean_cost, computing it (sequential sum on the device) if still unknown.
double graph_mean(const f2m_graph& g);

// Lambda layout conversion (host orig order <-> device position order).
void upload_lambda(const f2m_graph& g, const double* h_lambda, double* d_lam_pos);
void download_lambda(const f2m_graph& g, const double* d_lam_pos, double* h_lambda);

// dual.cu
// h_async (page-locked) != nullptr: the value is copied there asynchronously (valid after the
// stream's next synchronisation) and NaN is returned
double dual_objective_device(const f2m_graph& g, const double* d_lam_pos, int b, double* h_async = nullptr);
void initial_state_device(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam_pos,
                          int* h_err_async = nullptr);
struct SweepResult {
  int sweeps = 0;
  int converged = 0;
  double final_max_abs_delta = INFINITY;
  int out_buffer = 0;  // which of the two buffers holds the result
};
// threshold < 0: run exactly max_sweeps. defer_eps > 0 (threshold ignored): the threshold is
// defer_eps * mean_cost with mean_cost still unknown; the v5 kernel computes it (and g learns it).
SweepResult run_jacobi(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam0,
                       double* d_lam1, int max_sweeps, double threshold, double* d_record,
                       double defer_eps = 0.0);
void validate_engine(const f2m_engine_config& cfg);
// device time / sweeps of the most recent persistent sweep launch (f2m_last_sweep_kernel_ms)
void note_sweep_kernel(double ms, int sweeps);
// multi.cu: solve_duals on world_req GPUs from this host thread (EngineConfig::num_gpus > 1);
// d_lam_out: lambda in g's position order; rep: sweeps / converged / final max (no dual value)
void solve_duals_multi(const f2m_graph& g, const f2m_engine_config& cfg, int world_req, const double* d_init,
                       DBuf<double>& d_lam_out, f2m_convergence_report& rep);
// h_dual_async: see dual_objective_device (rep.dual_value is then left NaN for the caller)
void solve_duals_device(const f2m_graph& g, const f2m_engine_config& cfg, const double* d_init,
                        DBuf<double>& d_lam_out, f2m_convergence_report& rep, double* h_dual_async = nullptr);

// primal.cu
void extract_device(const f2m_graph& g, const double* d_lam_pos, double tol, double* d_x);
double objective_device(const f2m_graph& g, const double* d_x);
void verify_device(const f2m_graph& g, const double* d_x, double objective,
                   const double* d_lam_pos, f2m_verification& rep, int32_t* h_nodes,
                   double* h_sums, int32_t* h_vals, int64_t capacity, const double* dual_known = nullptr);
// objective + feasibility counts of the certified pipeline (no violation lists) with ONE
// synchronisation; dual: the dual objective (already known) for the gap
void certify_device(const f2m_graph& g, const double* d_x, double dual, double& objective, f2m_verification& rep);

// persistent sweep launch geometry (dual.cu)
int sweep_grid_ctas(int dev);
int sweep_block_threads();
size_t sweep_smem_limit(int dev);

// knn.cu
// xy: device pointer, or host pointer when xy_on_host (staged on the graph's own stream).
// start (nullable) is recorded on the graph's stream before any work (for device timing).
f2m_graph* knn_build_device(int n, const double* xy, bool xy_on_host, int rounded, int k, int dev,
                            cudaEvent_t start);

// ---------------------------------------------------------------- device helpers
// IEEE fp64 with no contraction: the reference is compiled without FMA (no -march), so
// every multiply-add below is an explicit rounded multiply followed by a rounded add.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Keeps the B+1 smallest values of a row in ascending s[0..B] (s starts at +inf): bubble val
// through the sorted list, branch-free. The kept multiset equals the reference's insertion
// (smallest_adjusted, dual.cpp:44-58) whatever the visiting order; a NaN val compares false
// everywhere and falls off the end, as `val < s[b]` rejects it in the reference.
template <int B>
__device__ __forceinline__ void topk_bubble(double (&s)[B + 1], double val) {
  // insertion into the ascending list with all compares against the OLD list (independent, so
  // they issue back to back): position i takes s[i-1] if val < s[i-1], val if s[i-1] <= val <
  // s[i], else keeps s[i]. Strict compares: val goes after equal elements, as a sequential
  // insertion would put it.
  bool c[B + 1];
#pragma unroll
  for (int i = 0; i <= B; ++i) c[i] = val < s[i];
#pragma unroll
  for (int i = B; i > 0; --i) s[i] = c[i - 1] ? s[i - 1] : (c[i] ? val : s[i]);
  s[0] = c[0] ? val : s[0];
}

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t state0, uint64_t draw_index) {
  // SplitMix64 (instance.hpp:54-60) is counter-based: the state before draw j (0-based) is
  // state0 + j*gamma, and next() first adds gamma.
  uint64_t z = state0 + (draw_index + 1ULL) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double splitmix64_double_at(uint64_t state0, uint64_t j) {
  return static_cast<double>(splitmix64_at(state0, j) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Polling loads are relaxed (an ld.acquire.gpu compiles to LDG.STRONG + CCTL.IVALL, an L1
// invalidation per poll); once the condition holds, one acquire fence orders what follows.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace f2mgpu

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
//                   global counter and poll the LL-published multipliers of lower neighbours.
//  k_gs_sweep       gauss_seidel_sweep (dual.cpp:175-192): one warp, nodes in id order.
//  k_dual_terms     dual_objective (dual.cpp:87-123): the terms in the reference's order; the
//                   2048/8192-chunk sequential sums come from seq_sums_device (seqsum.cu),
//                   bit-exact.
#include <chrono>
#include <climits>
#include <cstdlib>
#include <string>

#include <cstring>

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
  while (ld_relaxed_u32(bar) < target) {
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


// warp max of non-negative doubles (NaN skipped), as warp_max_nonneg below
__device__ __forceinline__ unsigned long long warp_max_nonneg_ap(double x) {
  const unsigned long long v = x == x ? (unsigned long long)__double_as_longlong(x) : 0ull;
  const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

// One TMA bulk prefetch of [p, p + bytes) into L2 (cp.async.bulk.prefetch.L2: 16-byte aligned
// start and size, so the range is widened to 16-byte boundaries). The streaming sweep form issues
// it a slice ahead per warp. (A row-ahead prefetch in the dense all-pairs form over-fills L2 —
// 4,736 warps x 64 KB rows — and re-fetches: 118 vs 92 us/sweep at n = 8,000, so it has none.)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  if (!bytes) return;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo)) : "memory");
}

// ---------------------------------------------------------------- all-pairs Jacobi sweep
// Complete graphs (build_knn_graph with k >= n-1, graph.cpp:175) whose costs are the points'
// distances: every cost is recomputed on the fly as distance() does it (instance.cpp:126-141:
// sqrt(dx*dx + dy*dy) without FMA, rounded mode floor(d + 0.5)) instead of streaming the
// n(n-1)/2-edge CSR — the FP64-pipe-bound variant of SURVEY §8(f). All points and the frozen
// multipliers sit in shared memory; one warp per node scans its n-1 partners (lane-strided) and
// the lanes' top lists are merged with shuffles. Same sweep/convergence protocol as k_gdp_sweep.
constexpr int kAllPairsThreads = 512;
#ifndef F2M_DENSE_THREADS
#define F2M_DENSE_THREADS 1024
#endif
constexpr int kDenseThreads = F2M_DENSE_THREADS;  // the streamed form wants memory-level parallelism
constexpr int kAllPairsMaxN = 8192;
// complete graphs with distance costs: 0 = the CSR kernels, 1 = recompute every cost from the
// points each sweep (FP64-bound), 2 = stream a once-computed distance matrix (default)
static std::atomic<int> g_allpairs_mode{2};

struct AllPairsArgs {
  int n;
  const double2* __restrict__ pts;  // position order
  const double* __restrict__ dense; // DENSE form: n x n distances in position order
  int rounded;
  double* lam0;
  double* lam1;
  double eta;
  int update;
  double threshold;
  int max_sweeps;
  double* record;
};

// DENSE form: the n x n distance matrix is computed once per graph (k_dense_distances, the same
// exact fp64 sequence) and every sweep streams row v (coalesced, 8 loads in flight per lane;
// L2-resident up to n ~ 3,900) instead of recomputing the square roots — HBM / L2-bound instead of
// FP64-bound.
// D[p][q] = distance(point p, point q) in position order, distance()'s exact sequence
// (instance.cpp:126-141: sqrt(dx*dx + dy*dy) without FMA, rounded mode floor(d + 0.5)) with dx taken
// from the row's point as the recompute form does; symmetric bit for bit.
__global__ void k_dense_distances(int n, const double2* __restrict__ pts, int rounded, double* __restrict__ d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * n) return;
  const int p = (int)(i / n), q = (int)(i - (int64_t)p * n);
  const double2 pv = pts[p], pu = pts[q];
  const double dx = dsub(pv.x, pu.x), dy = dsub(pv.y, pu.y);
  double c = __dsqrt_rn(dadd(dmul(dx, dx), dmul(dy, dy)));
  if (rounded) c = floor(dadd(c, 0.5));
  d[i] = c;
}

template <int B, bool DENSE>
__global__ void __launch_bounds__(DENSE ? kDenseThreads : kAllPairsThreads, 1) k_allpairs_sweep(AllPairsArgs a, SweepCtl* ctl) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[(DENSE ? kDenseThreads : kAllPairsThreads) / 32];
  __shared__ double s_gmax;
  double2* pts = reinterpret_cast<double2*>(smem);
  double* lam = DENSE ? reinterpret_cast<double*>(smem) : reinterpret_cast<double*>(pts + a.n);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (!DENSE)
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) pts[i] = a.pts[i];
  int sweep = 0;
  double gmax = INFINITY;
  bool converged = false;
  for (; sweep < a.max_sweeps; ++sweep) {
    const double* lin = (sweep & 1) ? a.lam1 : a.lam0;
    double* lout = (sweep & 1) ? a.lam0 : a.lam1;
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) lam[i] = __ldcg(lin + i);
    __syncthreads();
    double mx = 0.0;
    for (int v = blockIdx.x * nwarps + warp; v < a.n; v += gridDim.x * nwarps) {
      const double lv = lam[v];
      double s[B + 1];
#pragma unroll
      for (int i = 0; i <= B; ++i) s[i] = CUDART_INF;
      if (DENSE) {
        const double* __restrict__ row = a.dense + (size_t)v * a.n;
        int u = lane;
        for (; u + 224 < a.n; u += 256) {  // 8 coalesced row loads in flight per lane
          double c[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) c[q] = __ldcg(row + u + 32 * q);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const double z = dsub(dsub(c[q], lv), lam[u + 32 * q]);
            topk_bubble<B>(s, u + 32 * q != v ? z : CUDART_INF);
          }
        }
        for (; u < a.n; u += 32)
          if (u != v) topk_insert<B>(s, dsub(dsub(__ldcg(row + u), lv), lam[u]));
      } else {
        const double2 pv = pts[v];
        for (int u = lane; u < a.n; u += 32) {
          if (u == v) continue;
          const double2 pu = pts[u];
          const double dx = dsub(pv.x, pu.x), dy = dsub(pv.y, pu.y);
          double c = __dsqrt_rn(dadd(dmul(dx, dx), dmul(dy, dy)));
          if (a.rounded) c = floor(dadd(c, 0.5));
          topk_insert<B>(s, dsub(dsub(c, lv), lam[u]));
        }
      }
      warp_topk_merge<B>(s);
      if (lane == 0) {
        const double d = delta_of<B>(s, a.update);
        lout[v] = dadd(lv, dmul(a.eta, d));
        const double ad = fabs(d);
        mx = mx < ad ? ad : mx;
      }
    }
    const unsigned long long wm = warp_max_nonneg_ap(mx);
    if (lane == 0) red[warp] = __longlong_as_double((long long)wm);
    __syncthreads();
    if (threadIdx.x == 0) {
      double bm = 0.0;
      for (int w = 0; w < nwarps; ++w) bm = bm < red[w] ? red[w] : bm;
      if (blockIdx.x == 0) ctl->maxbits[(sweep + 1) % 3] = 0ull;
      atomicMax(&ctl->maxbits[sweep % 3], (unsigned long long)__double_as_longlong(bm));
      grid_barrier(&ctl->bar, (unsigned)(sweep + 1) * gridDim.x, &ctl->error);
      s_gmax = __longlong_as_double((long long)atomicAdd(&ctl->maxbits[sweep % 3], 0ull));
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

// Debug build only (-DF2M_WARP_PROFILE, tools/build_variant.sh): per-warp cycle accounting of the
// persistent sweep kernel — halo hand-off wait, boundary rows, interior rows, end-of-sweep barrier —
// summed over the sweeps of a launch and read back with f2m_debug_warp_profile. The product build
// compiles none of it.
#ifdef F2M_WARP_PROFILE
constexpr int kProfCtas = 160, kProfWarps = 32, kProfFields = 12;
__device__ unsigned long long g_wprof[kProfCtas][kProfWarps][kProfFields];
// per-CTA event clocks (SM clock64, comparable within a CTA) of sweeps [kTraceS0, kTraceS0 + 64):
// {sweep start, last boundary row published, halo staged (both sync warps), end-of-sweep barrier}
constexpr int kTraceS0 = 2000, kTraceN = 64;
__device__ unsigned long long g_strace[kProfCtas][kTraceN][4];
#define F2M_TRACE_EV(sw, f)                                                                 \
  do {                                                                                      \
    const int k_ = (sw) - kTraceS0;                                                         \
    if (k_ >= 0 && k_ < kTraceN && c < kProfCtas)                                           \
      atomicMax(&g_strace[c][k_][f], (unsigned long long)clock64());                        \
  } while (0)
// a volatile shared-memory read first: BAR.SYNC.DEFER_BLOCKING lets a warp run on until its next
// shared-memory access, so without it a clock read after a barrier is taken before the wait
#define F2M_PROF_T(var) \
  (void)*(volatile int*)&s_exit; \
  const long long var = clock64()
#define F2M_PROF_ADD(f, v) (prof[f] += (unsigned long long)(v))
#else
#define F2M_PROF_T(var)
#define F2M_PROF_ADD(f, v)
#define F2M_TRACE_EV(sw, f)
#endif

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

#ifndef F2M_RES_BATCH
#define F2M_RES_BATCH 4  // r02 A/B: 4 / 6 / 8 slots -> 100k 2.375 / 2.390 / 2.424 us, 200k 3.623 / 3.689 / 3.693
#endif
#ifndef F2M_STREAM_POLL
#define F2M_STREAM_POLL 4  // r02 A/B (4 vs 8): 2M 44.6 vs 44.4, 1M 22.1 vs 22.6, 400k 9.03 vs 9.46 us; spill-free
#endif
#ifndef F2M_STREAM_BATCH
#define F2M_STREAM_BATCH 6  // r02 A/B at 2M: 4 -> 52.0, 6 -> 46.5, 8 -> 49.1 us/sweep
#endif
#ifndef F2M_L2_PREFETCH_AHEAD
#define F2M_L2_PREFETCH_AHEAD 1
#endif
constexpr int kPrefetchAhead = F2M_L2_PREFETCH_AHEAD;  // streaming form: slices of L2 prefetch per warp
constexpr int kLamBufs = 8;     // convergence verdicts may lag the sweeps by up to 7
constexpr int kCmaxRing = 64;   // CTAs stay within ~16 sweeps of every helper (see core.cu)

// ---------------------------------------------------------------- persistent Jacobi sweep (LL)
// Partition-resident persistent kernel with no grid barrier.
//  * CTA c owns a contiguous, degree-balanced slice range; interior rows (all neighbours in the
//    CTA) first, boundary rows last. In resident mode the CTA's slot costs / local indices and
//    its multipliers live in shared memory for the whole solve (two lambda regions alternate).
//  * Inter-CTA traffic uses an LL ("low-latency") protocol: every published fp64 value travels
//    as two 8-byte words {tag:32 | half:32}, written with one relaxed 16-byte store and polled
//    with one relaxed 16-byte load. A word is single-copy atomic, so a matching tag in both
//    words proves the value is complete — no fences, no flags, one L2 trip from producer to
//    consumer (tools/microbench/pingpong.cu: 0.5-1.1 us vs 1.4-2.6 us for release/acquire flags).
//  * boundary node p of CTA c publishes lambda after sweep s at ll[(s+1)%kLLRing][boff[c] + p -
//    p0 - nint[c]] with tag s+1; halo readers poll exactly those entries (halo_pub).
//  * each CTA publishes its sweep max |delta| as an LL pair; a dedicated master CTA reduces them
//    in sweep order, applies max|delta| <= eps*mean_cost (dual.cpp:235) and publishes one
//    control word {stop:32 | verdicts:32}. A CTA starts sweep s+1 only once verdict s-7 exists,
//    so the result of the stopping sweep k (ring buffer (k+1)%8) is never overwritten; sweeps
//    after k are speculation and are discarded.
constexpr int kLLRing = 4;

__device__ __forceinline__ void st_ll(unsigned long long* p, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long hi = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)),
               "l"(hi | (b >> 32))
               : "memory");
}
__device__ __forceinline__ void ld_ll_raw(const unsigned long long* p, unsigned long long& w0,
                                          unsigned long long& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ bool ll_ok(unsigned long long w0, unsigned long long w1, unsigned tag) {
  return (unsigned)(w0 >> 32) == tag && (unsigned)(w1 >> 32) == tag;
}
__device__ __forceinline__ double ll_val(unsigned long long w0, unsigned long long w1) {
  return __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Sweep4Ctl {  // device-side control block (zeroed before each launch)
  unsigned long long word;  // {stop (k+1, 0 = running):32 | verdicts published:32}
  int abort;
  int sweeps;
  int converged;
  int out_buffer;
  double final_max;
};

struct Sweep4Args {
  int n;
  const int64_t* __restrict__ sptr;
  const int32_t* __restrict__ swidth;
  const int32_t* __restrict__ cta_lo;
  const int32_t* __restrict__ cta_int_hi;
  const int32_t* __restrict__ cta_nint;
  const int32_t* __restrict__ boff;
  const uint16_t* __restrict__ slidx;
  const double* __restrict__ scost;
  const int32_t* __restrict__ halo_off;
  const int32_t* __restrict__ halo;
  const int32_t* __restrict__ halo_pub;
  double* gl;                // full multipliers, kLamBufs contiguous buffers: sweep s writes
  size_t gstride;            // buffer (s+1)%8 at gl + ((s+1)%8)*gstride (no param-space indexing)
  unsigned long long* ll;    // [kLLRing][nb][2]
  int nb;
  unsigned long long* cmax;  // [kCmaxRing][G][2]
  double eta;
  int update;
  double threshold;
  int max_sweeps;
  double* record;
  int lam_stride;
  int halo_stride;           // ints of the halo LL-id region (max halo, multiple of 4)
  int lid4_stride;           // resident: packed local-index entries (ushort4) per CTA (max)
  const int32_t* __restrict__ sdest;     // v5: slot -> halo-last slot
  unsigned poll_ns;          // v5: sync-warp back-off between unproductive halo polls
  int runahead;              // v5: stage the next sweep's halo while this sweep computes
  int pair_rows;             // two lanes per boundary row (small graphs: <= 256 rows per CTA); selects
                             // the PAIR instantiation
  // deferred threshold (v5): defer_eps > 0 -> threshold = defer_eps * mean_cost, where the master
  // CTA computes mean_cost (sequential sum of cost[0..m) / m, graph.cpp:47-49) during the solve
  double defer_eps;
  const double* __restrict__ cost;
  int64_t m;
  const double* __restrict__ approx_sum;
  double* mean_out;
  // multi-GPU form (npeers > 0): this launch runs partition CTAs [cta_base, cta_base + gridDim.x -
  // 1) of g_total; every boundary multiplier and every CTA's sweep max is stored into all peers'
  // LL / max rings (peer memory), so each rank's master sees every CTA and issues the same verdicts
  int cta_base;
  int g_total;
  int npeers;
  unsigned long long* const* ll_peers;
  unsigned long long* const* cmax_peers;
  const uint32_t* __restrict__ ll_mask;  // [nb] ranks that read each boundary node
  int lam_ring;  // resident: multiplier regions in shared memory (2, or 8: the last 8 sweeps stay in
                 // shared memory and only the stopping sweep's result is written to gl at exit)
  int row_skip;  // resident head-first scans: per-row tail budgets (row_budget) in shared memory
};

constexpr uint64_t kWatchdogNs = 20ull * 1000000000ull;

// Per-CTA roles (k_gdp_sweep5):
//  * two sync warps run up to one sweep AHEAD of the compute warps: the halo of sweep s+1 is
//    polled and staged into the idle shared-memory region while sweep s is still computing, and
//    handed over through named barriers (no CTA-wide barrier between the roles);
//  * boundary rows (the only rows on the inter-CTA critical path) go first, one thread per row
//    (two lanes per row with a shuffle merge of their top-(B+1) lists on small graphs), and only
//    the warps that own them wait at the halo hand-off; the interior slices follow;
//  * one CTA barrier per sweep: the stop decision for sweep s+1 is taken before barrier B of s.

// warp max of non-negative doubles (|delta|) through their bit patterns (monotone for x >= 0):
// two REDUX ops instead of five 64-bit shuffle rounds. NaN is skipped like std::max(a, NaN) == a.
__device__ __forceinline__ unsigned long long warp_max_nonneg(double x) {
  const unsigned long long v = x == x ? (unsigned long long)__double_as_longlong(x) : 0ull;
  const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

// keep the B+1 smallest of two ascending lists (bitonic half-cleaner + sort of B+1 elements)
template <int B>
__device__ __forceinline__ void topk_merge(double (&s)[B + 1], const double (&o)[B + 1]) {
#pragma unroll
  for (int i = 0; i <= B; ++i) s[i] = o[B - i] < s[i] ? o[B - i] : s[i];
#pragma unroll
  for (int i = 0; i < B + 1; ++i) {
#pragma unroll
    for (int j = 0; j + 1 < B + 1 - i; ++j) {
      const bool sw = s[j + 1] < s[j];
      const double lo = sw ? s[j + 1] : s[j];
      s[j + 1] = sw ? s[j] : s[j + 1];
      s[j] = lo;
    }
  }
}

constexpr unsigned kPollBackoffNs = 64;
#ifndef F2M_POLL_NS
#define F2M_POLL_NS 64
#endif
constexpr unsigned kPollNs = F2M_POLL_NS;  // sync-warp back-off between unproductive halo polls

// Convergence master: a whole CTA on its own SM. Each round it reads the LL max |delta| of every
// CTA for a window of kMasterWindow sweeps in one pass (one L2 round trip for all of them), then
// thread 0 issues the verdicts for the complete sweeps in order (max|delta| <= eps*mean_cost,
// dual.cpp:235) and publishes {stop:32 | verdicts:32}. A one-sweep-per-round-trip master paces
// the whole grid at its own latency; the window takes it off the critical path.
constexpr int kMasterWindow = 16;

// CTA barrier of the master's verdict threads (all but warp 1 when warp 1 computes the mean)
__device__ __forceinline__ void master_sync(bool mean_warp_busy) {
  if (mean_warp_busy) named_sync(5, (int)blockDim.x - 32);
  else __syncthreads();
}

__device__ __noinline__ void sweep_master(const unsigned long long* __restrict__ cmax, int max_sweeps,
                                         double threshold, double* record, Sweep4Ctl* ctl, int G,
                                         double defer_eps, const double* __restrict__ cost, int64_t m,
                                         const double* __restrict__ approx_sum, double* mean_out) {
  __shared__ unsigned long long m_max[kMasterWindow];
  __shared__ int m_cnt[kMasterWindow];
  __shared__ int m_base, m_stop, m_quit;
  __shared__ double m_g;
  __shared__ int m_conv;
  __shared__ volatile int m_thr_ready;
  __shared__ double m_thr, m_lo, m_hi;
  __shared__ double m_tile[2][256];
  const int tid = threadIdx.x;
  if (tid == 0) {
    m_thr_ready = defer_eps > 0.0 ? 0 : 1;
    m_thr = threshold;
    if (defer_eps > 0.0) {
      // |sequential sum - any-order sum| <= 2 gamma_{m-1} * sum(c) for c >= 0; the mean's division
      // and the product with eps add 2u. delta is a generous over-estimate of the relative gap.
      const double u = 1.1102230246251565e-16;
      const double delta = 4.0 * ((double)m + 8.0) * u;
      const double est = m > 0 ? *approx_sum / (double)m : 0.0;
      m_lo = defer_eps * est * (1.0 - 2.0 * delta);
      m_hi = defer_eps * est * (1.0 + 2.0 * delta);
    }
  }
  if (tid == 0) {
    m_base = 0;
    m_stop = 0;
    m_quit = 0;
    m_g = INFINITY;
    m_conv = 0;
  }
  __syncthreads();
  if (defer_eps > 0.0 && (tid >> 5) == 1) {
    // graph.cpp:47-49: mean_cost = (sum over edges in order of cost) / m, one fp64 chain; lanes
    // stage 256-cost tiles (double-buffered) while lane 0 adds
    const int lane = tid & 31;
    double acc = 0.0;
    const int64_t ntiles = (m + 255) / 256;
    for (int i = lane; i < 256; i += 32) m_tile[0][i] = i < m ? cost[i] : 0.0;
    __syncwarp();
    for (int64_t t = 0; t < ntiles; ++t) {
      const int cur = t & 1;
      if (t + 1 < ntiles) {
        const int64_t b = (t + 1) * 256;
        for (int i = lane; i < 256; i += 32) m_tile[cur ^ 1][i] = b + i < m ? cost[b + i] : 0.0;
      }
      if (lane == 0) {
        const int cnt = (int)min64(256, m - t * 256);
        for (int i = 0; i < cnt; ++i) acc = dadd(acc, m_tile[cur][i]);
      }
      __syncwarp();
    }
    if (lane == 0) {
      const double mean = m > 0 ? __ddiv_rn(acc, (double)m) : 0.0;
      *mean_out = mean;
      m_thr = dmul(defer_eps, mean);  // cfg.eps * mean_cost (dual.cpp:221)
      __threadfence_block();
      m_thr_ready = 1;
    }
    return;
  }
  if (defer_eps > 0.0 && (tid >> 5) == 1) return;
  const uint64_t t_start = globaltimer_ns();
  uint64_t t_prog = t_start;
  for (;;) {
    const int base = m_base;
    if (tid < kMasterWindow) {
      m_max[tid] = 0ull;
      m_cnt[tid] = 0;
    }
    master_sync(defer_eps > 0.0);
    const int nthr = defer_eps > 0.0 ? (int)blockDim.x - 32 : (int)blockDim.x;
    const int rank = (defer_eps > 0.0 && tid >= 64) ? tid - 32 : tid;
    for (int e = rank; e < kMasterWindow * G; e += nthr) {
      const int w = e / G, cta = e - w * G, k = base + w;
      if (k >= max_sweeps) continue;
      unsigned long long w0, w1;
      ld_ll_raw(cmax + ((size_t)(k % kCmaxRing) * G + cta) * 2, w0, w1);
      if (ll_ok(w0, w1, (unsigned)k + 1)) {
        const double v = ll_val(w0, w1);
        atomicMax(&m_max[w], v == v ? (unsigned long long)__double_as_longlong(v) : 0ull);
        atomicAdd(&m_cnt[w], 1);
      }
    }
    master_sync(defer_eps > 0.0);
    if (tid == 0) {
      int k = base;
      unsigned stop = 0;
      for (int w = 0; w < kMasterWindow; ++w, ++k) {
        if (k >= max_sweeps || m_cnt[w] < G) break;
        const double g = __longlong_as_double((long long)m_max[w]);
        bool below;
        if (m_thr_ready) {
          below = g <= m_thr;
        } else if (g > m_hi) {
          below = false;  // above any threshold the exact mean can give
        } else if (g <= m_lo) {
          below = true;   // below any threshold the exact mean can give
        } else {
          break;          // undecidable until the exact mean is in: retry next round
        }
        if (record) record[k] = g;
        m_g = g;
        if (below) {
          m_conv = 1;
          stop = (unsigned)k + 1;
          ++k;
          break;
        }
        if (k == max_sweeps - 1) {
          stop = (unsigned)k + 1;
          ++k;
          break;
        }
      }
      const uint64_t now = globaltimer_ns();
      if (k > base || stop) {
        st_relaxed_u64(&ctl->word, ((unsigned long long)stop << 32) | (unsigned)k);
        t_prog = now;
      } else if (ld_relaxed(&ctl->abort) || now - t_prog > kWatchdogNs) {
        atomicExch(&ctl->abort, 1);
        stop = (unsigned)max(base, 1);
        st_relaxed_u64(&ctl->word, ((unsigned long long)stop << 32) | stop);
      }
      m_base = k;
      m_stop = (int)stop;
    }
    master_sync(defer_eps > 0.0);
    if (m_stop) break;
    if (m_base == base) __nanosleep(100);  // nothing new yet
  }
  if (tid == 0) {
    ctl->sweeps = m_stop;
    ctl->converged = m_conv;
    ctl->final_max = m_g;
    ctl->out_buffer = m_stop & 7;
  }
}

__device__ __forceinline__ void st_ll_sys(unsigned long long* p, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long hi = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)),
               "l"(hi | (b >> 32))
               : "memory");
}

// LL stores of the sweep kernel; in the multi-GPU form into every rank's ring (same offset,
// system scope: the readers are on other GPUs)
__device__ __forceinline__ void publish_ll(const Sweep4Args& a, unsigned long long* ring, int idx, double v,
                                           unsigned tag) {
  if (!a.npeers) {
    st_ll(ring + 2 * idx, v, tag);
    return;
  }
  // only the ranks whose CTAs read this boundary node (bit q of ll_mask[idx])
  const size_t off = (size_t)(ring - a.ll) + 2 * (size_t)idx;
  for (unsigned m = a.ll_mask[idx]; m; m &= m - 1) st_ll_sys(a.ll_peers[__ffs(m) - 1] + off, v, tag);
}
__device__ __forceinline__ void publish_cmax(const Sweep4Args& a, size_t off, double v, unsigned tag) {
  if (!a.npeers) {
    st_ll(a.cmax + off, v, tag);
    return;
  }
  for (int q = 0; q < a.npeers; ++q) st_ll_sys(a.cmax_peers[q] + off, v, tag);
}

// One row's scan over its slice's w slot columns (dual.cpp:33-61 smallest_adjusted for the lane's
// row): reduced costs (c - l_v) - l_u through the top-(B+1) list, KB slots per batch. Resident:
// costs and packed local indices from shared memory (l4 = this lane's packed-index column);
// streaming: both from global memory with evict-first loads.
template <int B, bool RES, int KB>
__device__ __forceinline__ void row_scan(double (&sv)[B + 1], double lv, const double* lam,
                                         const double* cst_s, const ushort4* l4, const double* __restrict__ gcost,
                                         const uint16_t* __restrict__ glid, int lb, int w) {
  int j = 0;
  for (; j + KB <= w; j += KB) {
    int li[KB];
    double cs[KB];
    if (RES) {
      static_assert(!RES || KB % 4 == 0, "packed indices: batches of 4");
#pragma unroll
      for (int g = 0; g < KB / 4; ++g) {
        const ushort4 q = l4[32 * ((j >> 2) + g)];
        li[4 * g] = q.x;
        li[4 * g + 1] = q.y;
        li[4 * g + 2] = q.z;
        li[4 * g + 3] = q.w;
      }
#pragma unroll
      for (int u = 0; u < KB; ++u) cs[u] = cst_s[lb + 32 * (j + u)];
    } else {
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        li[u] = __ldcs(glid + lb + 32 * (j + u));
        cs[u] = __ldcs(gcost + lb + 32 * (j + u));
      }
    }
#pragma unroll
    for (int u = 0; u < KB; ++u) topk_bubble<B>(sv, dsub(dsub(cs[u], lv), lam[li[u]]));
  }
  if (RES) {
    if (j < w) {  // tail: 1-3 slots of the last packed group
      const ushort4 q = l4[32 * (j >> 2)];
      const int lt[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (j + u < w) topk_bubble<B>(sv, dsub(dsub(cst_s[lb + 32 * (j + u)], lv), lam[lt[u]]));
    }
  } else {
    for (; j < w; ++j) topk_bubble<B>(sv, dsub(dsub(__ldcs(gcost + lb + 32 * j), lv), lam[__ldcs(glid + lb + 32 * j)]));
  }
}

#ifndef F2M_HEAD_SCAN
#define F2M_HEAD_SCAN 1
#endif
#ifndef F2M_BANK_LAYOUT
#define F2M_BANK_LAYOUT 1  // bank-aware initial slot order of the resident rows (layout_banks)
#endif
#ifndef F2M_LAYOUT_AUG
#define F2M_LAYOUT_AUG 1  // one-step augmenting paths in the warp layout
#endif
#ifdef F2M_HEAD_STATS  // debug build: repaired rows, printed at exit
__device__ unsigned long long g_head_stats[8];
#define F2M_HEAD_COUNT(i) atomicAdd(&g_head_stats[i], 1ull)
#else
#define F2M_HEAD_COUNT(i)
#endif

template <int MODE>
__device__ __forceinline__ bool tail_test(double v, double thr, double& tmin) {
  if (MODE == 1) {
    tmin = v < tmin ? v : tmin;
    return false;
  }
  return v < thr;
}

// An upper bound of the warp's largest non-negative double in one REDUX: the max of the high words,
// rounded up to the next high word (relative overestimate <= 2^-20)
__device__ __forceinline__ double warp_max_up(double x) {
  const unsigned hi = (unsigned)((unsigned long long)__double_as_longlong(x) >> 32);
  const unsigned m = __reduce_max_sync(0xffffffffu, x != 0.0 ? hi + 1u : 0u);
  return __longlong_as_double((long long)((unsigned long long)m << 32));
}

// Tail skipping (resident head-first scans, interior rows). The tail test of a row only has to prove that every
// tail slot's reduced cost stays >= the row's threshold s[B]. In exact arithmetic
// z_j - s[B] = (c_j - l_u) - OS_{B+1}(c_k - l_k) (l_v cancels), so from one sweep to the next it
// falls by at most 2 D, D = max |l_t - l_{t-1}| over the row's neighbours. A full tail scan at
// sweep s0 records the margin m = min_tail z - s[B]; while m - 2 (C_s - C_s0) stays above the
// rounding slack (C = running sum of per-sweep drift bounds of the CTA's own rows: an interior
// row's neighbours are all own rows, and the CTA's max |d| of each sweep is already reduced for the
// convergence test), every tail comparison of sweep s is false and only the head is evaluated.
// Boundary rows keep the plain tail test: with them skipping too (their halo's drift reduced by
// the sync warps or by the boundary warps), the exchange chain (staged -> published -> staged)
// got longer, 100k 2.09 -> 2.51 us per sweep (200k 2.98 -> 2.89; profiles/r02_ncu_sweep.md).
// Rounding: each computed z and s[B] is within 2.01 u (|c| + |l_v| + |l_u|) of exact, the
// multipliers stay below L0 + C (L0 = the CTA's largest |l| at the start), so a slack of
// 1e-12 (cmax + 2 L0 + 2 C) plus a 1e-9 relative allowance on C (its rounded accumulation over
// <= 1e6 sweeps) is rigorous; the result — which slots the tail compare finds below s[B] (none) —
// is exactly the one of the full scan, hence bit-identical deltas.
// The row's budget b = m (1 - 1e-9) + 2 C_s0 (1 - 1e-9) - 1e-12 (S0 + 2 C_s0), S0 = cmax + 2 L0;
// sweep s skips the tail iff b > 2 C_s (1 + 1e-9). The skip decision is warp-uniform (a warp's
// rows skip together or scan together: no divergent double path).
__device__ __forceinline__ double row_budget(double mn, double thr, double cc, double s0) {
  if (!(mn < CUDART_INF)) return CUDART_INF;  // no tail slots
  const double m = dsub(mn, thr);
  return dsub(dadd(dmul(m, 1.0 - 1e-9), dmul(2.0 - 2e-9, cc)), dmul(1e-12, dadd(s0, dmul(2.0, cc))));
}

// Resident row scan with a "head" of B+2 slots: the row's B+2 smallest slots of an earlier sweep,
// kept first in the row's shared-memory slot order. A row's smallest reduced costs almost never
// change membership from one sweep to the next (uniform 10k, per sweep: the top-(B+1) set of 0.09 %
// of rows changes, but only 0.014 % of rows see a slot from outside the previous top-(B+2) enter
// the top-(B+1); tools/head_stability.py), so:
//  * the head's B+2 reduced costs are sorted directly (a sorting network);
//  * every tail slot is only COMPARED with the (B+1)-th smallest head value: 2 DADD + 1 DSETP per
//    slot, no selects and no loop-carried chain, so the loads of all batches overlap;
//  * a row whose tail has a value below it is rescanned by the plain insertion (row_scan,
//    dual.cpp:44-58 smallest_adjusted) and row_repair moves its new B+2 smallest slots to the head.
// The kept multiset — the B+1 smallest reduced costs of the row — does not depend on the visiting
// order (reduced costs are never -0.0: costs are >= +0 and x - y = -0 only for x = -0), so s[B-1],
// s[B] and hence delta are bit-identical to the plain insertion over all slots.
// Returns true when the row must be rescanned. MODE 0: tail slots compared with the threshold;
// 1: also returns the smallest tail value in *mn (row skipping, below); 2: head only (the tail is
// proven to stay above the threshold).
template <int B, int MODE = 0>
__device__ __forceinline__ bool row_scan_head(double (&sv)[B + 2], double lv, const double* lam,
                                              const double* cst_s, const ushort4* l4, int lb, int w,
                                              double* mn = nullptr) {
  constexpr int H = B + 2;
  constexpr int HG = (H + 3) / 4;  // packed-index groups covering the head
  int li[4 * HG];
#pragma unroll
  for (int g = 0; g < HG; ++g) {
    const ushort4 q = l4[32 * g];
    li[4 * g] = q.x;
    li[4 * g + 1] = q.y;
    li[4 * g + 2] = q.z;
    li[4 * g + 3] = q.w;
  }
#pragma unroll
  for (int h = 0; h < H; ++h) sv[h] = dsub(dsub(cst_s[lb + 32 * h], lv), lam[li[h]]);
  auto cas = [&](int i, int k) {
    const bool sw = sv[k] < sv[i];
    const double lo = sw ? sv[k] : sv[i];
    sv[k] = sw ? sv[i] : sv[k];
    sv[i] = lo;
  };
  if (H == 4) {  // b = 2: the optimal 5-comparator network
    cas(0, 1);
    cas(2, 3);
    cas(0, 2);
    cas(1, 3);
    cas(1, 2);
  } else {  // odd-even transposition
#pragma unroll
    for (int r = 0; r < H; ++r) {
#pragma unroll
      for (int i = r & 1; i + 1 < H; i += 2) cas(i, i + 1);
    }
  }
  if (MODE == 2) return false;
  const double thr = sv[B];
  bool hit = false;
  double tmin = CUDART_INF;
  int j = H;
#define F2M_TAILV(jj, idx) tail_test<MODE>(dsub(dsub(cst_s[lb + 32 * (jj)], lv), lam[idx]), thr, tmin)
  if (H % 4) {  // tail slots of the last head group
#pragma unroll
    for (int u = 0; u < (4 - H % 4) % 4; ++u)
      if (j + u < w) hit |= F2M_TAILV(j + u, li[4 * HG - (4 - H % 4) + u]);
    j = 4 * HG;
  }
  for (; j + 4 <= w; j += 4) {
    const ushort4 q = l4[32 * (j >> 2)];
    const int lt[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) hit |= F2M_TAILV(j + u, lt[u]);
  }
  if (j < w) {  // 1-3 slots of the last packed group
    const ushort4 q = l4[32 * (j >> 2)];
    const int lt[3] = {q.x, q.y, q.z};
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (j + u < w) hit |= F2M_TAILV(j + u, lt[u]);
  }
#undef F2M_TAILV
  if (MODE == 1) {
    *mn = tmin;
    return tmin < thr;
  }
  return hit;
}

// Moves the row's K+1 smallest slots (values < s[K], then as many == s[K] as the list holds) to the
// head of its shared-memory slot order: a stable partition over the same frozen snapshot. Only
// the owning thread reads or writes a row's slots.
template <int K>
__device__ __forceinline__ void row_repair(const double (&sv)[K + 1], double lv, const double* lam, double* cst_s,
                                           ushort4* l4, int lb, int w) {
  uint16_t* lid = reinterpret_cast<uint16_t*>(l4);
  F2M_HEAD_COUNT(1);
  const double thr = sv[K];
  int needeq = 0;
#pragma unroll
  for (int i = 0; i <= K; ++i) needeq += !(sv[i] < thr);
  int cnt = 0;
  for (int j = 0; j < w && cnt <= K; ++j) {
    const int xj = 128 * (j >> 2) + (j & 3);
    const uint16_t ij = lid[xj];
    const double cj = cst_s[lb + 32 * j];
    const double v = dsub(dsub(cj, lv), lam[ij]);
    bool take = v < thr;
    if (!take && v == thr && needeq > 0) {
      take = true;
      --needeq;
    }
    if (take) {
      if (j != cnt) {
        const int xc = 128 * (cnt >> 2) + (cnt & 3);
        lid[xj] = lid[xc];
        cst_s[lb + 32 * j] = cst_s[lb + 32 * cnt];
        lid[xc] = ij;
        cst_s[lb + 32 * cnt] = cj;
      }
      ++cnt;
    }
  }
}

#ifndef F2M_SKIP_WARP
#define F2M_SKIP_WARP 1
#endif
// One resident row through the head-first scan (and, with tail skipping, its budget): the B+1
// smallest reduced costs into sv.
template <int B, bool RES, int KB>
__device__ __forceinline__ void row_head_first(double (&sv)[B + 1], double lv, const double* lam, double* cst_s,
                                               ushort4* l4, const double* __restrict__ gcost,
                                               const uint16_t* __restrict__ glid, int lb, int w, bool skip,
                                               double* budp, double cc, double sk0) {
  double hv[B + 2];
  bool rescan;
  if (skip) {
    bool ok = *budp > dmul(2.000000002, cc);
#if F2M_SKIP_WARP  // warp-uniform: the warp's rows skip together or scan together (no divergence)
    ok = __all_sync(__activemask(), ok);
#endif
    if (ok) {
      F2M_HEAD_COUNT(6);
      row_scan_head<B, 2>(hv, lv, lam, cst_s, l4, lb, w);
      rescan = false;
    } else {
      F2M_HEAD_COUNT(7);
      double mn;
      rescan = row_scan_head<B, 1>(hv, lv, lam, cst_s, l4, lb, w, &mn);
      *budp = rescan ? -CUDART_INF : row_budget(mn, hv[B], cc, sk0);
    }
  } else {
    rescan = row_scan_head<B>(hv, lv, lam, cst_s, l4, lb, w);
  }
  if (rescan) {
#pragma unroll
    for (int i = 0; i <= B + 1; ++i) hv[i] = CUDART_INF;
    row_scan<B + 1, RES, KB>(hv, lv, lam, cst_s, l4, gcost, glid, lb, w);
    row_repair<B + 1>(hv, lv, lam, cst_s, l4, lb, w);
  }
#pragma unroll
  for (int i = 0; i <= B; ++i) sv[i] = hv[i];
}

// Initial slot order of one row (resident form, kernel setup): its B+2 smallest reduced costs at
// the initial multipliers (lam0: own + staged halo) go to columns 0..B+1, the head of
// row_scan_head. sl = {slot offset, width, packed-index offset} of the row's slice, l = its lane.
__device__ __noinline__ void layout_head(int B, double* cst_s, ushort4* lid4, int4 sl, int l, double lv,
                                         const double* lam0) {
  uint16_t* lid = reinterpret_cast<uint16_t*>(lid4);
  const int w = sl.y;
  auto ix = [&](int k) { return (sl.z + 32 * (k >> 2) + l) * 4 + (k & 3); };
  for (int h = 0; h < B + 2 && h < w; ++h) {  // selection: the smallest of columns h.. to column h
    int best = h;
    double bv = dsub(dsub(cst_s[sl.x + l + 32 * h], lv), lam0[lid[ix(h)]]);
    for (int k = h + 1; k < w; ++k) {
      const double v = dsub(dsub(cst_s[sl.x + l + 32 * k], lv), lam0[lid[ix(k)]]);
      if (v < bv) {
        bv = v;
        best = k;
      }
    }
    if (best != h) {
      const uint16_t t = lid[ix(h)];
      lid[ix(h)] = lid[ix(best)];
      lid[ix(best)] = t;
      const double c = cst_s[sl.x + l + 32 * h];
      cst_s[sl.x + l + 32 * h] = cst_s[sl.x + l + 32 * best];
      cst_s[sl.x + l + 32 * best] = c;
    }
  }
}

// Bank-aware column order of one half-slice (the 16 rows one half-warp scans together; a 64-bit
// shared-memory load is served per half-warp, one 8-byte word per bank pair = local index mod 16).
// Column by column, each row takes the first of its remaining slots whose multiplier word falls in
// a bank pair no earlier row of the half-warp uses in that column, or is the same word (a
// broadcast). A row with no such slot tries a one-step augmenting path: a bank pair it can reach
// whose single user can move to a free pair. Otherwise it keeps its slot (a conflict). Head columns
// (0..B+1) only permute among themselves. Order only: the scans' results do not depend on it.
// Rows [l0, l0 + nrows) of the slice sl.
__device__ __noinline__ void layout_banks(int B, double* cst_s, ushort4* lid4, int4 sl, int l0, int nrows) {
  uint16_t* lid = reinterpret_cast<uint16_t*>(lid4);
  const int w = sl.y, H = w > B + 1 ? B + 2 : 0;
  auto ix = [&](int l, int k) { return (sl.z + 32 * (k >> 2) + l) * 4 + (k & 3); };
  auto swap_cols = [&](int l, int j, int k) {
    const int xj = ix(l, j), xk = ix(l, k);
    const uint16_t t = lid[xj];
    lid[xj] = lid[xk];
    lid[xk] = t;
    const double c = cst_s[sl.x + l + 32 * j];
    cst_s[sl.x + l + 32 * j] = cst_s[sl.x + l + 32 * k];
    cst_s[sl.x + l + 32 * k] = c;
  };
  for (int j = 0; j < w; ++j) {
    const int hi = j < H ? H : w;
    unsigned used = 0, shared = 0;  // bank pairs in use / used by more than one row (a broadcast)
    uint16_t word[16];
    int8_t owner[16];
    for (int l = l0; l < l0 + nrows; ++l) {
      int pick = -1;
      for (int k = j; k < hi; ++k) {
        const uint16_t q = lid[ix(l, k)];
        if (!((used >> (q & 15)) & 1u) || word[q & 15] == q) {
          pick = k;
          break;
        }
      }
      if (pick < 0) {  // one-step augmenting path
        for (int k = j; k < hi && pick < 0; ++k) {
          const int b = lid[ix(l, k)] & 15;
          if ((shared >> b) & 1u) continue;
          const int o = owner[b];
          for (int k2 = j + 1; k2 < hi; ++k2) {
            const uint16_t q2 = lid[ix(o, k2)];
            if (!((used >> (q2 & 15)) & 1u)) {
              swap_cols(o, j, k2);  // the owner moves to the free pair
              used |= 1u << (q2 & 15);
              word[q2 & 15] = q2;
              owner[q2 & 15] = (int8_t)o;
              used &= ~(1u << b);
              pick = k;
              break;
            }
          }
        }
      }
#ifdef F2M_HEAD_STATS
      F2M_HEAD_COUNT(j < H ? 4 : 5);
      if (pick < 0) F2M_HEAD_COUNT(j < H ? 2 : 3);
#endif
      if (pick < 0) pick = j;
      if (pick != j) swap_cols(l, j, pick);
      const uint16_t q = lid[ix(l, j)];
      const int b = q & 15;
      if ((used >> b) & 1u) {
        shared |= 1u << b;  // a broadcast (or a conflict: the pair stays with its first word)
      } else {
        used |= 1u << b;
        word[b] = q;
        owner[b] = (int8_t)l;
      }
    }
  }
}

// layout_banks run by a whole warp (same greedy, same result): the lanes scan one row's remaining
// candidate columns at once (lane i: column j + i) and a ballot picks the first acceptable one, so
// a (row, column) step costs one shared-memory load per lane instead of a serial scan. Needs
// w <= 32 (the caller falls back to layout_banks otherwise). wd: this warp's 16-word scratch.
__device__ __forceinline__ void layout_banks_warp(int B, double* cst_s, ushort4* lid4, int4 sl, int l0, int nrows,
                                               uint16_t* wd) {
  uint16_t* lid = reinterpret_cast<uint16_t*>(lid4);
  const int lane = threadIdx.x & 31;
  const int w = sl.y, H = w > B + 1 ? B + 2 : 0;
  auto ix = [&](int l, int k) { return (sl.z + 32 * (k >> 2) + l) * 4 + (k & 3); };
  auto swap_cols = [&](int l, int j, int k) {  // lane 0 only
    const int xj = ix(l, j), xk = ix(l, k);
    const uint16_t t = lid[xj];
    lid[xj] = lid[xk];
    lid[xk] = t;
    const double c = cst_s[sl.x + l + 32 * j];
    cst_s[sl.x + l + 32 * j] = cst_s[sl.x + l + 32 * k];
    cst_s[sl.x + l + 32 * k] = c;
  };
  for (int j = 0; j < w; ++j) {
    const int hi = j < H ? H : w;
    unsigned used = 0, shared = 0;
    unsigned long long owner = 0;  // 4 bits per bank pair: the row (l - l0) using it
    for (int l = l0; l < l0 + nrows; ++l) {
      const int k = j + lane;
      const bool in = k < hi;
      const int q = in ? lid[ix(l, k)] : 0, b = q & 15;
      const bool ok = in && (!((used >> b) & 1u) || wd[b] == q);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      int pick = m ? j + __ffs(m) - 1 : -1;
      if (pick < 0 && F2M_LAYOUT_AUG) {  // one-step augmenting path, candidates in column order
        const unsigned cand = __ballot_sync(0xffffffffu, in);
        for (unsigned cm = cand; cm && pick < 0; cm &= cm - 1) {
          const int kk = j + __ffs(cm) - 1;
          const int bb = __shfl_sync(0xffffffffu, b, kk - j);
          if ((shared >> bb) & 1u) continue;
          const int o = l0 + (int)((owner >> (4 * bb)) & 15);
          const int k2 = j + 1 + lane;
          const bool in2 = k2 < hi;
          const int q2 = in2 ? lid[ix(o, k2)] : 0;
          const unsigned m2 = __ballot_sync(0xffffffffu, in2 && !((used >> (q2 & 15)) & 1u));
          if (m2) {
            const int k2s = j + __ffs(m2);
            const int q2s = __shfl_sync(0xffffffffu, q2, k2s - (j + 1));
            if (lane == 0) {
              swap_cols(o, j, k2s);
              wd[q2s & 15] = (uint16_t)q2s;
            }
            __syncwarp();
            used |= 1u << (q2s & 15);
            owner = (owner & ~(15ull << (4 * (q2s & 15)))) | ((unsigned long long)(o - l0) << (4 * (q2s & 15)));
            used &= ~(1u << bb);
            pick = kk;
          }
        }
      }
#ifdef F2M_HEAD_STATS
      if (lane == 0) {
        F2M_HEAD_COUNT(j < H ? 4 : 5);
        if (pick < 0) F2M_HEAD_COUNT(j < H ? 2 : 3);
      }
#endif
      if (pick < 0) pick = j;
      const int qp = __shfl_sync(0xffffffffu, q, pick - j);
      if (lane == 0 && pick != j) swap_cols(l, j, pick);
      const int bq = qp & 15;
      if ((used >> bq) & 1u) {
        shared |= 1u << bq;
      } else {
        used |= 1u << bq;
        if (lane == 0) wd[bq] = (uint16_t)qp;
        owner = (owner & ~(15ull << (4 * bq))) | ((unsigned long long)(l - l0) << (4 * bq));
      }
      __syncwarp();
    }
  }
}

template <int B, bool RES, int NT, bool PAIR>
__global__ void __launch_bounds__(NT, 1) k_gdp_sweep5(Sweep4Args a, Sweep4Ctl* ctl) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[2][NT / 32];
  __shared__ int s_stop[2];
  __shared__ volatile int s_done;  // sweeps completed by the compute warps
  __shared__ volatile int s_exit;
  __shared__ unsigned long long s_word;
  __shared__ uint16_t s_lw[NT / 32][16];  // layout_banks_warp scratch, one per warp
  __shared__ unsigned long long s_scale[2];  // tail skipping: max |cost|, max |l0| (own + halo)
  // CTAs 0..G-1 own the partition; the last CTA of the launch (alone on its SM) is the master.
  // Multi-GPU: this launch's CTAs are the partition CTAs cta_base.. of g_total.
  const int G = a.npeers ? a.g_total : (int)gridDim.x - 1;
  const int c = (int)blockIdx.x + (a.npeers ? a.cta_base : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int sync0 = nwarps - 2, ncw = nwarps - 2;
  if (blockIdx.x == gridDim.x - 1) {
    sweep_master(a.cmax, a.max_sweeps, a.threshold, a.record, ctl, G, a.defer_eps, a.cost, a.m, a.approx_sum,
                 a.mean_out);
    return;
  }
  const int cthreads = ncw * 32;
  // slots per batch of the row scans: shared-memory scans keep few loads in flight (fewer live
  // registers, less rematerialisation), the streaming form's global loads are bounded by its
  // 64-register budget at 1024 threads (A/B figures at the macro definitions)
  constexpr int kBatch = RES ? F2M_RES_BATCH : F2M_STREAM_BATCH;
  constexpr bool kHead = RES && F2M_HEAD_SCAN;  // head-first row scans (row_scan_head)
  constexpr bool kSkipT = kHead && F2M_BANK_LAYOUT && F2M_ROW_SKIP;
  // (not in the small-graph PAIR form: 10k 1.75 -> 1.79 us/sweep with it, few interior rows per CTA)
  const bool kSkip = kSkipT && !PAIR && a.row_skip;
  const int s_lo = a.cta_lo[c], s_hi = a.cta_lo[c + 1], s_int = a.cta_int_hi[c];
  const int p0 = s_lo * 32;
  const int own = max(0, min(s_hi * 32, a.n) - p0);
  const int nint = a.cta_nint[c];
  const int bo = a.boff[c] - nint;
  const int bstart = min((s_int - s_lo) * 32, own);  // boundary phase: local [bstart, own)
  const int nbnd = own - bstart;
  // boundary row of this thread (per batch of cthreads rows): the rotation starts at the first
  // warp with the fewest interior slices, so boundary work lands on the least-loaded warps
  const int brow = (tid - ((s_int - s_lo) % ncw) * 32 + cthreads) % cthreads;
  // only the warps that own boundary rows (and the sync warps) meet at the halo hand-off; the
  // others go straight to their interior rows. Two lanes per boundary row when the CTA has few of
  // them (small graphs: at 10k the boundary chain dominates and idle lanes are plentiful; at 100k+
  // the interior rows need the lanes)
  const bool pair_rows = RES && PAIR && 2 * nbnd <= cthreads;
  const int bthreads = pair_rows ? 2 * nbnd : nbnd;  // threads (in rotated order) with boundary work
  const bool own_bar = bthreads <= cthreads;
  const int halo_bar = own_bar ? 64 + 32 * ((bthreads + 31) / 32) : cthreads + 64;
  const bool in_halo_bar = !own_bar || (brow & ~31) < bthreads;
  const int h0 = a.halo_off[c], nh = a.halo_off[c + 1] - h0;
  const int64_t slot0 = a.sptr[s_lo];
  const int nslots = (int)(a.sptr[s_hi] - slot0);
  double* regA = reinterpret_cast<double*>(smem);
  double* regB = regA + (RES ? a.lam_stride : 0);
  // resident: lam_ring regions; sweep s reads region s % ring and writes region (s + 1) % ring
  const int ring = RES ? a.lam_ring : 1;
  auto region = [&](int i) { return regA + (size_t)(RES ? (ring == 8 ? (i & 7) : (i & 1)) : 0) * a.lam_stride; };
  const bool gl_each_sweep = !RES || ring != 8;  // else the result goes to gl once, at exit
  int* halo_s = reinterpret_cast<int*>(regA + (RES ? ring : 1) * a.lam_stride);
  double* cst_s = reinterpret_cast<double*>(halo_s + a.halo_stride);
  // resident local indices, packed 4 slots per lane: slice t's slot (j, lane) is component j % 4 of
  // lid4[slc[t].z + 32 (j / 4) + lane] — one 8-byte load per lane per 4 slots instead of four 2-byte
  // loads (widths are padded to a multiple of 4 for this array only; the padding is never read)
  ushort4* lid4 = reinterpret_cast<ushort4*>(cst_s + (RES ? nslots : 0));
  const int nlid4 = RES ? a.lid4_stride : 0;
  // per-slice {slot offset, width, packed-index offset} of this CTA: no global loads on the sweep
  // path. The 16-byte alignment is computed on the offset from `smem` so the compiler keeps the
  // shared address space (a uintptr_t round trip turned these into generic LD.E loads)
  const size_t slc_off = ((size_t)(reinterpret_cast<unsigned char*>(lid4 + nlid4) - smem) + 15) & ~size_t(15);
  int4* slc = reinterpret_cast<int4*>(smem + slc_off);
  // tail skipping: one budget per own row after the slice table (host: + 16 + 8 max_local bytes)
  double* bud = reinterpret_cast<double*>(smem + ((slc_off + 16 * (size_t)(s_hi - s_lo) + 15) & ~size_t(15)));
  const double* __restrict__ gcost = a.scost + slot0;
  const uint16_t* __restrict__ glid = a.slidx + slot0;
  for (int i = tid; i < nh; i += blockDim.x) halo_s[i] = a.halo_pub[h0 + i];
  if (tid == 0) {  // <= ~60 slices per CTA in the resident regime
    s_scale[0] = s_scale[1] = 0ull;
    int z = 0;
    for (int i = 0; i < s_hi - s_lo; ++i) {
      const int w = a.swidth[s_lo + i];
      slc[i] = make_int4((int)(a.sptr[s_lo + i] - slot0), w, z, 0);
      z += 32 * ((w + 3) >> 2);
    }
  }
  if (RES) {
    __syncthreads();  // slice table in place
    const int ns = s_hi - s_lo;
    for (int i = tid; i < nslots; i += blockDim.x) {  // rows stored own-first, halo-last
      const int d = (int)(a.sdest[slot0 + i] - slot0);
      cst_s[d] = gcost[i];
      int t0 = 0, t1 = ns;  // slice holding destination slot d
      while (t1 - t0 > 1) {
        const int mid = (t0 + t1) >> 1;
        if (slc[mid].x <= d) t0 = mid; else t1 = mid;
      }
      const int r = d - slc[t0].x, j = r >> 5;
      reinterpret_cast<uint16_t*>(lid4)[(size_t)(slc[t0].z + 32 * (j >> 2) + (r & 31)) * 4 + (j & 3)] = glid[i];
    }
    for (int i = tid; i < own; i += blockDim.x) regA[i] = a.gl[p0 + i];
    if (kHead && F2M_BANK_LAYOUT) {
      // initial slot order: heads at the initial multipliers (halo staged here once), then
      // bank-aware columns
      for (int i = tid; i < nh; i += blockDim.x) regA[own + i] = __ldcg(a.gl + a.halo[h0 + i]);
      __syncthreads();
      if (kSkip) {  // the rounding-slack scale of the tail budgets
        double cm = 0.0, lm = 0.0;
        for (int i = tid; i < nslots; i += blockDim.x)  // padding slots (+inf) give z = +inf exactly
          if (fabs(cst_s[i]) < CUDART_INF) cm = fmax(cm, fabs(cst_s[i]));
        for (int i = tid; i < own + nh; i += blockDim.x) lm = fmax(lm, fabs(regA[i]));
        for (int i = tid; i < own; i += blockDim.x) bud[i] = -CUDART_INF;  // first sweep: full scans
        const unsigned long long cw = warp_max_nonneg(cm), lw = warp_max_nonneg(lm);
        if (lane == 0) {
          atomicMax(&s_scale[0], cw);
          atomicMax(&s_scale[1], lw);
        }
      }
      for (int lp = tid; lp < own; lp += blockDim.x) layout_head(B, cst_s, lid4, slc[lp >> 5], lp & 31, regA[lp], regA);
      __syncthreads();
      // one warp per half-slice (one thread when a slice is wider than 32 slots)
      for (int hs = warp; hs < 2 * ns; hs += nwarps) {
        const int l0 = 16 * (hs & 1), nrows = min(16, own - 32 * (hs >> 1) - l0);
        if (nrows <= 0) continue;
        if (slc[hs >> 1].y <= 32) layout_banks_warp(B, cst_s, lid4, slc[hs >> 1], l0, nrows, s_lw[warp]);
        else if (lane == 0) layout_banks(B, cst_s, lid4, slc[hs >> 1], l0, nrows);
      }
    }
  }
  if (tid == 0) {
    s_word = 0ull;
    s_stop[0] = s_stop[1] = -1;
    s_done = 0;
    s_exit = 0;
  }
  __syncthreads();

  if (warp >= sync0) {
    // ---- sync warps: stage the halo of sweep s (LL tag s; sweep 0: the initial multipliers)
    const int sw = warp - sync0;
    // halo entries per lane per poll round: 8 in the resident form; the streaming form's
    // 64-register budget (1024 threads) may favour fewer loads in flight
    constexpr int kPB = RES ? 8 : F2M_STREAM_POLL;
    for (int s = 0;; ++s) {
      const int need = (RES && a.runahead) ? s - 1 : s;  // the region being filled is no longer read
      while (s_done < need && !s_exit) __nanosleep(32);
      if (s_exit) break;
      double* lam = region(s);
      const double* gin = (a.gl + (size_t)(s & 7) * a.gstride);
      const unsigned long long* llin = a.ll + (size_t)(s % kLLRing) * a.nb * 2;
      const uint64_t t0 = globaltimer_ns();
      bool quit = false;
      for (int base = sw * 32; base < nh && !quit; base += 64 * kPB) {
        unsigned pend = 0;
#pragma unroll
        for (int b = 0; b < kPB; ++b)
          if (base + lane + 64 * b < nh) pend |= 1u << b;
        if (s == 0) {
          double v[kPB];
#pragma unroll
          for (int b = 0; b < kPB; ++b)
            if (pend & (1u << b)) v[b] = __ldcg(gin + a.halo[h0 + base + lane + 64 * b]);
#pragma unroll
          for (int b = 0; b < kPB; ++b)
            if (pend & (1u << b)) lam[own + base + lane + 64 * b] = v[b];
          continue;
        }
        int it = 0;
        while (__any_sync(0xffffffffu, pend != 0)) {
          const unsigned pend_before = pend;
          unsigned long long w0[kPB], w1[kPB];
#pragma unroll
          for (int b = 0; b < kPB; ++b)
            if (pend & (1u << b)) ld_ll_raw(llin + 2 * halo_s[base + lane + 64 * b], w0[b], w1[b]);
#pragma unroll
          for (int b = 0; b < kPB; ++b)
            if ((pend & (1u << b)) && ll_ok(w0[b], w1[b], (unsigned)s)) {
              lam[own + base + lane + 64 * b] = ll_val(w0[b], w1[b]);
              pend &= ~(1u << b);
            }
          // back off while nothing arrives: a spinning poller floods the SM's memory pipe that
          // the compute warps' shared-memory loads share
          if (__all_sync(0xffffffffu, pend == pend_before) && a.poll_ns) __nanosleep(a.poll_ns);
          if ((++it & 15) == 0) {
            int q = 0;
            if (lane == 0) {
              const unsigned long long w = ld_relaxed_u64(&ctl->word);
              s_word = w;
              q = (w >> 32) != 0 || ld_relaxed(&ctl->abort) || s_exit;
              if (!q && globaltimer_ns() - t0 > kWatchdogNs) {
                atomicExch(&ctl->abort, 1);
                q = 1;
              }
            }
            if (__shfl_sync(0xffffffffu, q, 0)) {
              pend = 0;
              quit = true;
            }
          }
        }
      }
      __syncwarp();
      // hand-off on a hardware barrier (compute warps sleep in bar.sync, no spinning); two ids
      // alternate so the run-ahead arrival for s+1 can never be counted towards sweep s
      if (lane == 0) F2M_TRACE_EV(s, 2);
      named_arrive(3 + (s & 1), halo_bar);
      if (sw == 0 && lane == 0) s_word = ld_relaxed_u64(&ctl->word);
    }
    return;
  }

  // ---- compute warps. Boundary rows (the only rows other CTAs read) first: the halo of sweep s
  // was published early in the neighbours' sweep s-1 (they too start with their boundary rows),
  // so it is normally staged already; publish, then the interior rows overlap the neighbours'
  // next exchange.
#ifdef F2M_WARP_PROFILE
  unsigned long long prof[kProfFields] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
  int s_stop_final = -1;
  // tail skipping: running sum of the per-sweep drift bounds (identical in every thread)
  double c_own = 0.0, sk0 = 0.0;
  if (kSkip) sk0 = dadd(__longlong_as_double((long long)s_scale[0]), dmul(2.0, __longlong_as_double((long long)s_scale[1])));
  for (int s = 0;; ++s) {
    F2M_PROF_T(t0);
    if (tid == 0) F2M_TRACE_EV(s, 0);
    double* lam = region(s);
    double* lam_next = RES ? region(s + 1) : ((s & 1) ? regA : regB);
    const double* gin = (a.gl + (size_t)(s & 7) * a.gstride);
    double* gout = (a.gl + (size_t)((s + 1) & 7) * a.gstride);
    if (!RES) {
      for (int i = tid; i < own; i += cthreads) lam[i] = __ldcg(gin + p0 + i);
      named_sync(2, cthreads);
    }
    double mx = 0.0;
    if (kSkip && s > 0) {
      // own rows: |l_s - l_{s-1}| <= eta |d| (1 + 2u) + u |l_s| (the CTA max |d| of sweep s-1)
      const double dm = warp_max_up(lane < ncw ? red[(s - 1) & 1][lane] : 0.0);
      c_own = dadd(c_own, dadd(dmul(fabs(a.eta), dm), dmul(1e-15, dadd(sk0, c_own))));
    }
    if (in_halo_bar) named_sync(3 + (s & 1), halo_bar);  // halo of sweep s staged
    F2M_PROF_T(t1);
    F2M_PROF_ADD(0, t1 - t0);
    unsigned long long* llout = a.ll + (size_t)((s + 1) % kLLRing) * a.nb * 2;
    if (pair_rows) {
      // two lanes per boundary row (even / odd slots), one shuffle merge
      if ((brow & ~31) < 2 * nbnd) {
        const int node = brow >> 1, half = brow & 1;
        double sv[B + 1];
#pragma unroll
        for (int i = 0; i <= B; ++i) sv[i] = CUDART_INF;
        int lp = 0, p = 0;
        double lv = 0.0;
        if (node < nbnd) {
          lp = bstart + node;
          p = p0 + lp;
          const int4 sw2 = slc[(p >> 5) - s_lo];
          const int lb = sw2.x + (p & 31);
          const int w = sw2.y;
          const uint16_t* lidr = reinterpret_cast<const uint16_t*>(lid4 + sw2.z + (p & 31));
          lv = lam[lp];
          for (int jj = half; jj < w; jj += 8) {
            int li[4];
            double cs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool ok = jj + 2 * u < w;
              const int jx = ok ? jj + 2 * u : 0;
              const int idx = lb + 32 * jx;
              li[u] = lidr[128 * (jx >> 2) + (jx & 3)];
              cs[u] = cst_s[idx];
              if (!ok) {
                li[u] = lp;
                cs[u] = CUDART_INF;
              }
            }
            double lu[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) lu[u] = lam[li[u]];
#pragma unroll
            for (int u = 0; u < 4; ++u) topk_bubble<B>(sv, dsub(dsub(cs[u], lv), lu[u]));
          }
        }
        double ov[B + 1];
#pragma unroll
        for (int i = 0; i <= B; ++i) ov[i] = __shfl_xor_sync(0xffffffffu, sv[i], 1);
        topk_merge<B>(sv, ov);
        if (node < nbnd && half == 0) {
          const double d = delta_of<B>(sv, a.update);
          const double nl = dadd(lv, dmul(a.eta, d));
          if (lp >= nint) publish_ll(a, llout, bo + lp, nl, (unsigned)s + 1);
          if (gl_each_sweep) gout[p] = nl;
          lam_next[lp] = nl;
          const double ad = fabs(d);
          mx = mx < ad ? ad : mx;
        }
      }
    } else {
      for (int base = 0; base < nbnd; base += cthreads) {
        if (base + (brow & ~31) >= nbnd) break;  // warp-uniform: no row for this warp
        const int node = base + brow;
        if (node < nbnd) {
          const int lp = bstart + node, p = p0 + lp;
          const int4 sw2 = slc[(p >> 5) - s_lo];
          const int lb = sw2.x + (p & 31);
          const int w = sw2.y;
          double sv[B + 1];
#pragma unroll
          for (int i = 0; i <= B; ++i) sv[i] = CUDART_INF;
          const double lv = lam[lp];
          F2M_PROF_T(ta);
          // the warp's 32 lanes are the 32 rows of one boundary slice (bstart is slice-aligned):
          // one width, so the interior rows' batches apply without predication
          if (kHead && w > B + 1) {
            row_head_first<B, RES, kBatch>(sv, lv, lam, cst_s, lid4 + sw2.z + (p & 31), gcost, glid, lb, w, false,
                                           nullptr, 0.0, 0.0);
          } else {
            row_scan<B, RES, kBatch>(sv, lv, lam, cst_s, lid4 + sw2.z + (p & 31), gcost, glid, lb, w);
          }
          F2M_PROF_T(tb);
          const double d = delta_of<B>(sv, a.update);
          const double nl = dadd(lv, dmul(a.eta, d));
          if (lp >= nint) publish_ll(a, llout, bo + lp, nl, (unsigned)s + 1);
          if (gl_each_sweep) gout[p] = nl;
          if (RES) lam_next[lp] = nl;
          const double ad = fabs(d);
          mx = mx < ad ? ad : mx;
          F2M_PROF_T(tc);
          F2M_PROF_ADD(8, ta - t1);
          F2M_PROF_ADD(9, tb - ta);
          F2M_PROF_ADD(10, tc - tb);
        }
      }
    }
    F2M_PROF_T(t2);
    if (lane == 0 && nbnd > 0 && in_halo_bar) F2M_TRACE_EV(s, 1);
    F2M_PROF_ADD(1, t2 - t1);
    // interior slices: one thread per node (throughput-bound phase)
    for (int sl = s_lo + warp; sl < s_int; sl += ncw) {
      if (!RES && lane == 0) {
        // this warp's slice F2M_L2_PREFETCH_AHEAD slices from now, or (near the end of the sweep)
        // its first slice of the next sweep: the slot arrays are the same every sweep
        const int nx = sl + kPrefetchAhead * ncw < s_int ? sl + kPrefetchAhead * ncw : s_lo + warp;
        const int4 q = slc[nx - s_lo];
        prefetch_l2(gcost + q.x, (unsigned)q.y * 32u * 8u);
        prefetch_l2(glid + q.x, (unsigned)q.y * 32u * 2u);
      }
      const int p = sl * 32 + lane;
      if (p >= a.n) continue;
      const int lp = p - p0;
      const int4 sw2 = slc[sl - s_lo];
      const int lb = sw2.x + lane;
      const int w = sw2.y;
      const double lv = lam[lp];
      double sv[B + 1];
#pragma unroll
      for (int i = 0; i <= B; ++i) sv[i] = CUDART_INF;
      if (kHead && w > B + 1) {
        row_head_first<B, RES, kBatch>(sv, lv, lam, cst_s, lid4 + sw2.z + lane, gcost, glid, lb, w, kSkip, bud + lp,
                                       c_own, sk0);
      } else {
        row_scan<B, RES, kBatch>(sv, lv, lam, cst_s, lid4 + sw2.z + lane, gcost, glid, lb, w);
      }
      const double d = delta_of<B>(sv, a.update);
      const double nl = dadd(lv, dmul(a.eta, d));
      if (gl_each_sweep) gout[p] = nl;
      if (RES) lam_next[lp] = nl;
      const double ad = fabs(d);
      mx = mx < ad ? ad : mx;
    }
    F2M_PROF_T(t3);
    F2M_PROF_ADD(2, t3 - t2);
    {
      const unsigned long long wm = warp_max_nonneg(mx);
      if (lane == 0) red[s & 1][warp] = __longlong_as_double((long long)wm);
    }
    if (warp == 0 && lane == 0) {
      // stop decision for sweep s+1 (it overwrites glam[(s+2)%8]): verdict s-7 must be in
      unsigned long long w = s_word;
      const uint64_t t0 = globaltimer_ns();
      int it = 0;
      const int s1 = s + 1;
      for (;;) {
        const unsigned stop = (unsigned)(w >> 32), done = (unsigned)w;
        if (stop) break;
        if (s1 >= a.max_sweeps) {  // budget spent: stop after this sweep; the master picks k
          w = (unsigned long long)(unsigned)s1 << 32;
          break;
        }
        if ((int)done >= s1 - kLamBufs + 1) break;
        if ((++it & 63) == 0 && (ld_relaxed(&ctl->abort) || globaltimer_ns() - t0 > kWatchdogNs)) {
          atomicExch(&ctl->abort, 1);
          w = (unsigned long long)(unsigned)s1 << 32;
          break;
        }
        w = ld_relaxed_u64(&ctl->word);
      }
      s_word = w;
      s_stop[s & 1] = (w >> 32) ? (int)(w >> 32) - 1 : -1;
    }
    named_sync(2, cthreads);  // [B]
#ifdef F2M_WARP_PROFILE
    if (tid == 0) {
      (void)*(volatile int*)&s_exit;
      F2M_TRACE_EV(s, 3);
    }
#endif
    F2M_PROF_T(t4);
    F2M_PROF_ADD(3, t4 - t3);
    F2M_PROF_ADD(4, 1);
    if (warp == ncw - 1) {  // the CTA max goes out from the warp with the least boundary work
      const unsigned long long bm = warp_max_nonneg(lane < ncw ? red[s & 1][lane] : 0.0);
      if (lane == 0) {
        publish_cmax(a, ((size_t)(s % kCmaxRing) * G + c) * 2, __longlong_as_double((long long)bm), (unsigned)s + 1);
        s_done = s + 1;
      }
    }
    if (s_stop[s & 1] >= 0) {
      s_stop_final = s_stop[s & 1];
      break;
    }
  }
#ifdef F2M_WARP_PROFILE
  if (lane == 0 && c < kProfCtas && warp < kProfWarps) {
    // static work of this warp: interior slices and their slot columns, boundary rows (per sweep)
    int isl = 0, icol = 0;
    for (int sl = s_lo + warp; sl < s_int; sl += ncw) { ++isl; icol += slc[sl - s_lo].y; }
    prof[5] = isl;
    prof[6] = icol;
    // width of this warp's boundary slice (0: no boundary rows)
    prof[7] = (!pair_rows && (brow & ~31) < nbnd) ? slc[((p0 + bstart + (brow & ~31)) >> 5) - s_lo].y : 0;
    for (int f = 0; f < kProfFields; ++f) g_wprof[c][warp][f] = prof[f];
  }
#endif
  if (!gl_each_sweep && s_stop_final >= 0) {
    // the stopping sweep k's result (shared-memory region (k + 1) % 8, never overwritten: a CTA runs
    // at most sweep k + 7, see the verdict lag) goes to gl buffer (k + 1) % 8, where the host reads it
    const double* res = region(s_stop_final + 1);
    double* gdst_out = a.gl + (size_t)((s_stop_final + 1) & 7) * a.gstride + p0;
    for (int i = tid; i < own; i += cthreads) gdst_out[i] = res[i];
  }
  if (tid == 0) s_exit = 1;
#ifdef F2M_HEAD_STATS
  if (tid == 0 && c == 0)
    printf("head stats: repaired rows %llu; layout conflicts head %llu / %llu, tail %llu / %llu; tail skipped %llu, "
           "scanned %llu\n", g_head_stats[1], g_head_stats[2], g_head_stats[4], g_head_stats[3], g_head_stats[5],
           g_head_stats[6], g_head_stats[7]);
#endif
}

template <int B, bool RES, int NT, bool PAIR>
static void launch_sweep5(const Sweep4Args& a, Sweep4Ctl* ctl, int ctas, size_t smem, cudaStream_t s) {
  auto fn = k_gdp_sweep5<B, RES, NT, PAIR>;
  F2M_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {(void*)&a, (void*)&ctl};
  F2M_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(ctas), dim3(NT), args, smem, s));
}

#ifndef F2M_PAIR_ROWS_PER_CTA
#define F2M_PAIR_ROWS_PER_CTA 256
#endif
constexpr int kPairRowsPerCta = F2M_PAIR_ROWS_PER_CTA;  // two lanes per boundary row up to this many rows per CTA
#ifndef F2M_STREAMING_THREADS
#define F2M_STREAMING_THREADS 1024
#endif
#ifndef F2M_RES_THREADS
#define F2M_RES_THREADS 768  // r02 A/B with packed indices: 768 / 896 / 1024 -> 100k 2.265 / 2.269 / 2.701 us
#endif
constexpr int kResidentThreads = F2M_RES_THREADS;
constexpr int kStreamingThreads = F2M_STREAMING_THREADS;

// Resident (smem) layout: 768 threads per CTA (22 compute warps + 2 sync warps, 80 registers) with
// the boundary-first sweep order: at 100k 3.18 us/sweep vs 3.40 (640), 3.48 (832), 3.73 (704),
// 3.66 (1024) — more warps hide more latency until ptxas' register budget (65536 / threads)
// serialises each row's load chain (640 was best with the interior-first order). The streaming
// layout keeps 1024 threads for memory-level parallelism.
template <bool RES, int NT, bool PAIR>
static void dispatch_sweep5_b(int b, const Sweep4Args& a, Sweep4Ctl* ctl, int ctas, size_t smem, cudaStream_t s) {
  switch (b) {
    case 1: launch_sweep5<1, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 2: launch_sweep5<2, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 3: launch_sweep5<3, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 4: launch_sweep5<4, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 5: launch_sweep5<5, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 6: launch_sweep5<6, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    case 7: launch_sweep5<7, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
    default: launch_sweep5<8, RES, NT, PAIR>(a, ctl, ctas, smem, s); break;
  }
}

// the three product forms: resident with two lanes per boundary row (small graphs), resident with
// one thread per boundary row, streaming (slots read from global memory every sweep)
static void dispatch_sweep5(const Topology& t, int b, const Sweep4Args& a, Sweep4Ctl* ctl, int ctas, cudaStream_t s) {
  if (t.resident && a.pair_rows) dispatch_sweep5_b<true, kResidentThreads, true>(b, a, ctl, ctas, t.smem_bytes, s);
  else if (t.resident) dispatch_sweep5_b<true, kResidentThreads, false>(b, a, ctl, ctas, t.smem_bytes, s);
  else dispatch_sweep5_b<false, kStreamingThreads, false>(b, a, ctl, ctas, t.smem_bytes, s);
}

size_t sweep_smem_limit(int dev) {
  const cudaDeviceProp& p = device_props(dev);
  // headroom for the kernels' static shared memory (v5: ~4.5 KB incl. the master's tiles)
  return p.sharedMemPerBlockOptin > 8192 ? p.sharedMemPerBlockOptin - 8192 : 0;
}

static double g_last_sweep_ms = 0.0;
static std::string g_last_sweep_desc = "none";
static int g_last_sweep_count = 0;

template <int B>
static void launch_sweep(const SweepArgs& a, SweepCtl* ctl, int ctas, cudaStream_t s) {
  void* args[] = {(void*)&a, (void*)&ctl};
  F2M_CUDA(cudaLaunchCooperativeKernel((const void*)k_gdp_sweep<B>, dim3(ctas), dim3(kSweepThreads),
                                       args, 0, s));
}

// F2M_SWEEP_VARIANT=1 (or the older F2M_SWEEP_V1=1) forces the grid-barrier kernel for A/B
// measurements; it is also used whenever the per-CTA local index space does not fit (!t.v2).
static int g_variant = -1;

static int sweep_variant(const Topology& t) {
  if (g_variant < 0) {
    g_variant = 5;
    if (const char* e = std::getenv("F2M_SWEEP_VARIANT"))
      if (std::atoi(e) == 1) g_variant = 1;
    if (const char* e = std::getenv("F2M_SWEEP_V1"))
      if (e[0] == '1') g_variant = 1;
  }
  return t.v2 ? g_variant : 1;
}

static bool use_v1(const Topology& t) { return sweep_variant(t) == 1; }

SweepResult run_jacobi(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam0,
                       double* d_lam1, int max_sweeps, double threshold, double* d_record,
                       double defer_eps) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  SweepResult r;
  if (max_sweeps <= 0) return r;
  if (defer_eps > 0.0 && (g.mean_known || sweep_variant(t) == 1)) {
    threshold = defer_eps * graph_mean(g);  // host fp64 product, no FMA: == cfg.eps * mean_cost
    defer_eps = 0.0;
  }
  cudaEvent_t e0, e1;
  F2M_CUDA(cudaEventCreate(&e0));
  F2M_CUDA(cudaEventCreate(&e1));
  int error = 0, sweeps = 0, converged = 0, outbuf = 0;
  double final_max = INFINITY;
  const int ap_mode = g_allpairs_mode.load();
  if (g.allpairs && ap_mode != 0 && t.n <= kAllPairsMaxN) {
    const double2* pts = g.pts_pos.get();
    const bool dense = ap_mode == 2;
    if (dense && !g.dense.get()) {  // once per graph (n^2 doubles: 537 MB at the 8,192 cap)
      g.dense.alloc((size_t)t.n * t.n, s);
      k_dense_distances<<<grid_for((int64_t)t.n * t.n, 256), 256, 0, s>>>(t.n, pts, g.rounded, g.dense.get());
      launched("dense_distances");
    }
    DBuf<SweepCtl> ctl(1, s);
    F2M_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(SweepCtl), s));
    AllPairsArgs ap;
    ap.n = t.n;
    ap.pts = pts;
    ap.dense = dense ? g.dense.get() : nullptr;
    ap.rounded = g.rounded;
    ap.lam0 = d_lam0;
    ap.lam1 = d_lam1;
    ap.eta = cfg.eta;
    ap.update = cfg.update;
    ap.threshold = defer_eps > 0.0 ? defer_eps * graph_mean(g) : threshold;
    ap.max_sweeps = max_sweeps;
    ap.record = d_record;
    const size_t smem = (size_t)t.n * ((dense ? 0 : sizeof(double2)) + sizeof(double));
    // one row per warp; the dense form spreads its rows over every SM (up to 32 warps each)
    const int sms = sweep_grid_ctas(t.dev);
    const int nt = dense ? std::min(kDenseThreads, std::max(64, 32 * ((t.n + sms - 1) / sms))) : kAllPairsThreads;
    const int wpc = nt / 32;
    const int ctas = std::min(sms, std::max(1, (t.n + wpc - 1) / wpc));
    g_last_sweep_desc = "k_allpairs_sweep<b=" + std::to_string(cfg.b) + (dense ? ", dense" : ", recompute") +
                        "> (" + std::to_string(ctas) + " CTAs x " + std::to_string(nt) + ", " +
                        (dense ? "distance matrix streamed, " : "costs recomputed from the points, ") +
                        std::to_string(smem) + " B smem/CTA)";
    F2M_CUDA(cudaEventRecord(e0, s));
    SweepCtl* ctlp = ctl.get();
    void* args[] = {(void*)&ap, (void*)&ctlp};
    auto launch = [&](const void* fn) {
      F2M_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      F2M_CUDA(cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(nt), args, smem, s));
    };
    switch (cfg.b) {
#define F2M_AP(BB)                                                                                        \
  case BB:                                                                                                \
    launch(dense ? (const void*)k_allpairs_sweep<BB, true> : (const void*)k_allpairs_sweep<BB, false>);  \
    break;
      F2M_AP(1) F2M_AP(2) F2M_AP(3) F2M_AP(4) F2M_AP(5) F2M_AP(6) F2M_AP(7)
      default: launch(dense ? (const void*)k_allpairs_sweep<8, true> : (const void*)k_allpairs_sweep<8, false>); break;
#undef F2M_AP
    }
    launched("allpairs_sweep");
    F2M_CUDA(cudaEventRecord(e1, s));
    SweepCtl h;
    F2M_CUDA(cudaMemcpyAsync(&h, ctl.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    error = h.error;
    sweeps = h.sweeps;
    converged = h.converged;
    final_max = h.final_max;
    outbuf = (h.sweeps & 1) ? 1 : 0;
  } else if (use_v1(t)) {
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
    g_last_sweep_desc = "k_gdp_sweep<b=" + std::to_string(cfg.b) + "> (grid barrier, " + std::to_string(t.sweep_ctas) + " CTAs)";
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
    error = h.error;
    sweeps = h.sweeps;
    converged = h.converged;
    final_max = h.final_max;
    outbuf = (h.sweeps & 1) ? 1 : 0;
  } else {
    const int G = t.sweep_ctas;
    DBuf<double> ring((size_t)kLamBufs * std::max(t.n, 1), s);
    DBuf<Sweep4Ctl> ctl(1, s);
    const int nb = std::max(t.nboundary, 1);
    DBuf<unsigned long long> ll((size_t)kLLRing * nb * 2, s);
    DBuf<unsigned long long> cmax((size_t)kCmaxRing * G * 2, s);
    // tags restart at 1 every launch: stale words from an earlier launch must not match
    F2M_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(Sweep4Ctl), s));
    F2M_CUDA(cudaMemsetAsync(ll.get(), 0, ll.bytes(), s));
    F2M_CUDA(cudaMemsetAsync(cmax.get(), 0, cmax.bytes(), s));
    Sweep4Args a;
    a.n = t.n;
    a.sptr = t.sptr.get();
    a.swidth = t.swidth.get();
    a.cta_lo = t.cta_lo.get();
    a.cta_int_hi = t.cta_int_hi.get();
    a.cta_nint = t.cta_nint.get();
    a.boff = t.boff.get();
    a.slidx = t.slidx.get();
    a.scost = g.scost.get();
    a.halo_off = t.halo_off.get();
    a.halo = t.halo.get();
    a.halo_pub = t.halo_pub.get();
    a.gl = ring.get();
    a.gstride = (size_t)std::max(t.n, 1);
    if (t.n > 0) F2M_CUDA(cudaMemcpyAsync(ring.get(), d_lam0, sizeof(double) * t.n, cudaMemcpyDeviceToDevice, s));
    a.ll = ll.get();
    a.nb = nb;
    a.sdest = t.sdest.get();
    a.poll_ns = kPollNs;
    a.runahead = 1;
    DBuf<double> mean_out(1, s);
    a.defer_eps = defer_eps;
    a.cost = g.cost.get();
    a.m = t.m;
    a.approx_sum = g.approx_sum.get();
    a.mean_out = mean_out.get();
    // boundary rows first, only their warps meet at the halo hand-off; on small graphs (<= 256
    // rows per CTA: the boundary chain dominates, lanes are idle) two lanes per boundary row.
    // Measured: 10k 2.51 -> 2.09 us/sweep with pairs; at 100k / 200k pairs cost 6 %.
    a.pair_rows = t.n <= kPairRowsPerCta * G ? 1 : 0;
    a.cmax = cmax.get();
    a.eta = cfg.eta;
    a.update = cfg.update;
    a.threshold = threshold;
    a.max_sweeps = max_sweeps;
    a.record = d_record;
    a.lam_stride = (int)((((size_t)t.max_local * sizeof(double) + 15) & ~size_t(15)) / sizeof(double));
    a.lam_ring = t.resident ? t.lam_ring : 2;
    a.row_skip = t.resident ? t.row_skip : 0;
    a.halo_stride = (t.max_halo + 3) & ~3;
    a.lid4_stride = (int)t.max_cta_lid4;
    a.cta_base = 0;
    a.g_total = G;
    a.npeers = 0;
    a.ll_peers = nullptr;
    a.cmax_peers = nullptr;
    a.ll_mask = nullptr;
    F2M_CUDA(cudaEventRecord(e0, s));
    {  // + 1 CTA: the convergence master
      g_last_sweep_desc = "k_gdp_sweep5<b=" + std::to_string(cfg.b) +
                          (t.resident ? ", resident, " + std::to_string(kResidentThreads)
                                      : ", streaming, " + std::to_string(kStreamingThreads)) +
                          "> (persistent: " + std::to_string(G) +
                          " partition CTAs + 1 convergence-master CTA, LL halo exchange, " +
                          std::to_string(t.smem_bytes) + " B smem/CTA" +
                          (a.pair_rows ? ", two lanes per boundary row)" : ")");
      dispatch_sweep5(t, cfg.b, a, ctl.get(), G + 1, s);
      launched("gdp_sweep5");
    }
    F2M_CUDA(cudaEventRecord(e1, s));
    // control block and deferred mean through page-locked scratch: one synchronisation
    static_assert(sizeof(Sweep4Ctl) <= 16 * sizeof(int64_t), "pinned scratch layout");
    int64_t* ps = pinned_scratch();
    F2M_CUDA(cudaMemcpyAsync(ps + 32, ctl.get(), sizeof(Sweep4Ctl), cudaMemcpyDeviceToHost, s));
    if (defer_eps > 0.0) F2M_CUDA(cudaMemcpyAsync(ps + 48, mean_out.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    Sweep4Ctl h;
    std::memcpy(&h, ps + 32, sizeof(h));
    double hmean = 0.0;
    if (defer_eps > 0.0) std::memcpy(&hmean, ps + 48, sizeof(double));
    if (defer_eps > 0.0 && !h.abort) {
      g.mean_cost = hmean;  // bit-identical to sequential_mean (same chain, same order)
      g.mean_known = true;
    }
    error = h.abort;
    sweeps = h.sweeps;
    converged = h.converged;
    final_max = h.final_max;
    outbuf = h.out_buffer;
    if (t.n > 0)
      F2M_CUDA(cudaMemcpyAsync(d_lam1, a.gl + (size_t)outbuf * a.gstride, sizeof(double) * t.n,
                               cudaMemcpyDeviceToDevice, s));
    outbuf = 1;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_last_sweep_ms = ms;
  g_last_sweep_count = sweeps;
  if (error) throw Error(F2M_E_TIMEOUT, "gdp sweep kernel: synchronisation watchdog fired");
  r.sweeps = sweeps;
  r.converged = converged;
  r.final_max_abs_delta = final_max;
  r.out_buffer = outbuf;
  return r;
}

// ---------------------------------------------------------------- init (make_initial_state)
template <int B>
__global__ void __launch_bounds__(256) k_init_local_midpoint(
    int n, const int32_t* __restrict__ perm, const int32_t* __restrict__ iperm,
    const int32_t* __restrict__ deg, const int64_t* __restrict__ sptr,
    const int32_t* __restrict__ scol, const double* __restrict__ scost, double* lam,
    unsigned long long* ll, int* counter, int* err) {
  // node p's final multiplier is published once as an LL pair {1:32 | half:32} x 2 (see st_ll):
  // a reader's single 16-byte poll both detects completion and returns the value (no flag, no
  // fence, one L2 round trip)
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
        unsigned long long w0, w1;
        for (;;) {
          ld_ll_raw(ll + 2 * (int64_t)q, w0, w1);
          if (ll_ok(w0, w1, 1u)) break;
          if (globaltimer_ns() - t0 > 20ull * 1000000000ull) {
            atomicExch(err, 1);
            break;
          }
        }
        other = ll_val(w0, w1);
      }
      // ge.cost - lv - other with lv = lambda[v] = 0 (dual.cpp:43)
      topk_insert<B>(s, dsub(dsub(c, 0.0), other));
    }
    warp_topk_merge<B>(s);
    if (lane == 0) {
      const double val = d > B ? dmul(0.5, dadd(s[B - 1], s[B])) : 0.0;
      st_ll(ll + 2 * (int64_t)p, val, 1u);
      lam[p] = val;
    }
  }
}

// make_initial_state (dual.cpp:194-208) with one thread per node: warps claim 32 consecutive
// node ids at a time (ids start in order), each lane scans its node's row and waits (LL poll) only
// for the neighbours with lower ids, exactly the values the reference's in-order pass has already
// written. The kept multiset of the b+1 smallest is the warp form's, so lambda_0 is bit-identical;
// the dependency chain (DAG depth ~26 at 100k) no longer queues behind one warp per node.
template <int B>
__global__ void __launch_bounds__(256) k_init_thread(
    int n, const int32_t* __restrict__ perm, const int32_t* __restrict__ iperm,
    const int32_t* __restrict__ deg, const int64_t* __restrict__ sptr,
    const int32_t* __restrict__ scol, const double* __restrict__ scost, double* lam,
    unsigned long long* ll, int* counter, int* err) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const int v = base + lane;
    if (v >= n) continue;
    const int p = perm[v];
    const int d = deg[p];
    const int64_t rb = sptr[p >> 5] + (p & 31);
    double sv[B + 1];
#pragma unroll
    for (int i = 0; i <= B; ++i) sv[i] = CUDART_INF;
    // slots in chunks of 4: the LL words of all lower-id neighbours of a chunk are polled together
    // (one L2 round trip per round, not one per neighbour)
    for (int j0 = 0; j0 < d; j0 += 4) {
      int q[4];
      double c[4], other[4];
      unsigned pend = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        other[u] = 0.0;  // lambda of a higher-numbered (or the same) node is still 0
        c[u] = CUDART_INF;
        q[u] = 0;
        if (j0 + u < d) {
          q[u] = scol[rb + (int64_t)(j0 + u) * 32];
          c[u] = scost[rb + (int64_t)(j0 + u) * 32];
          if (iperm[q[u]] < v) pend |= 1u << u;
        }
      }
      const uint64_t t0 = pend ? globaltimer_ns() : 0;
      while (pend) {
        unsigned long long w0[4], w1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pend & (1u << u)) ld_ll_raw(ll + 2 * (int64_t)q[u], w0[u], w1[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((pend & (1u << u)) && ll_ok(w0[u], w1[u], 1u)) {
            other[u] = ll_val(w0[u], w1[u]);
            pend &= ~(1u << u);
          }
        if (pend && globaltimer_ns() - t0 > 20ull * 1000000000ull) {
          atomicExch(err, 1);
          break;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < d) topk_insert<B>(sv, dsub(dsub(c[u], 0.0), other[u]));  // ge.cost - lv - other, lv = 0
    }
    const double val = d > B ? dmul(0.5, dadd(sv[B - 1], sv[B])) : 0.0;
    st_ll(ll + 2 * (int64_t)p, val, 1u);
    lam[p] = val;
  }
}

#ifndef F2M_INIT_THREAD
#define F2M_INIT_THREAD 1
#endif

template <int B>
static void launch_init(const f2m_graph& g, double* d_lam, unsigned long long* ll, int* counter, int* err) {
  const Topology& t = *g.topo;
  if (F2M_INIT_THREAD) {
    // persistent: every thread of the grid is resident, so a claimed id's lower neighbours are held
    // by running threads (ids are claimed in increasing order)
    const int blocks = std::max(1, std::min<int>(grid_for(t.n, 256), device_props(t.dev).multiProcessorCount * 8));
    k_init_thread<B><<<blocks, 256, 0, t.stream>>>(t.n, t.perm.get(), t.iperm.get(), t.deg.get(), t.sptr.get(),
                                                  t.scol.get(), g.scost.get(), d_lam, ll, counter, err);
    launched("init_thread");
    return;
  }
  // 4 CTAs (32 warps) per SM: measured 0.14 ms at 100k vs 0.23 ms with 8 (fewer warps spinning
  // on the id-order frontier, less contention on the claim counter)
  const int blocks = std::max(1, std::min<int>(grid_for((int64_t)t.n * 32, 256),
                                               device_props(t.dev).multiProcessorCount * 4));
  k_init_local_midpoint<B><<<blocks, 256, 0, t.stream>>>(t.n, t.perm.get(), t.iperm.get(), t.deg.get(),
                                                        t.sptr.get(), t.scol.get(), g.scost.get(), d_lam,
                                                        ll, counter, err);
  launched("init_local_midpoint");
}

void initial_state_device(const f2m_graph& g, const f2m_engine_config& cfg, double* d_lam_pos, int* h_err_async) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  if (t.n == 0) return;
  F2M_CUDA(cudaMemsetAsync(d_lam_pos, 0, sizeof(double) * t.n, s));
  if (cfg.init != 0) return;  // kZero
  DBuf<unsigned long long> ll((size_t)2 * t.n, s);
  DBuf<int> flags(2, s);
  F2M_CUDA(cudaMemsetAsync(ll.get(), 0, ll.bytes(), s));
  F2M_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int) * 2, s));
  unsigned long long* llp = ll.get();
  int* counter = flags.get();
  int* err = flags.get() + 1;
  switch (cfg.b) {
    case 1: launch_init<1>(g, d_lam_pos, llp, counter, err); break;
    case 2: launch_init<2>(g, d_lam_pos, llp, counter, err); break;
    case 3: launch_init<3>(g, d_lam_pos, llp, counter, err); break;
    case 4: launch_init<4>(g, d_lam_pos, llp, counter, err); break;
    case 5: launch_init<5>(g, d_lam_pos, llp, counter, err); break;
    case 6: launch_init<6>(g, d_lam_pos, llp, counter, err); break;
    case 7: launch_init<7>(g, d_lam_pos, llp, counter, err); break;
    default: launch_init<8>(g, d_lam_pos, llp, counter, err); break;
  }
  if (h_err_async) {  // pinned: the caller reads it after its next synchronisation
    F2M_CUDA(cudaMemcpyAsync(h_err_async, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    return;
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

// phase 1 of jacobi_sweep (dual.cpp:138-152) alone: every node's delta from the frozen lambda,
// one warp per node (the pooled jacobi_sweep overload's delta scratch)
template <int B>
__global__ void k_all_deltas(int n, const int32_t* __restrict__ deg, const int64_t* __restrict__ sptr,
                             const int32_t* __restrict__ scol, const double* __restrict__ scost,
                             const double* lam, int update, double* __restrict__ out) {
  const int p = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (p >= n) return;
  const double r = row_delta_warp<B>(p, deg[p], sptr, scol, scost, lam, update);
  if ((threadIdx.x & 31) == 0) out[p] = r;
}

// ---------------------------------------------------------------- dual objective
// Terms of the dual objective in the reference's accumulation order: lambda[v] for the node
// chunks (dual.cpp:96-100) and min(v_e, 0) for the edge chunks, v_e = (c - l_u) - l_v
// (dual.cpp:101-109). Adding +0.0 for v_e >= 0 is exact: an edge chunk's running value is +0.0
// or a negative non-zero sum, both unchanged by +0.0.
__global__ void __launch_bounds__(256) k_dual_terms(int n, int64_t m, const int32_t* __restrict__ perm,
                                                    const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                                    const double* __restrict__ cost, const double* __restrict__ lam,
                                                    double* __restrict__ terms) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    terms[i] = lam[perm[i]];
  } else if (i < n + m) {
    const int64_t e = i - n;
    const double x = dsub(dsub(cost[e], lam[perm[eu[e]]]), lam[perm[ev[e]]]);
    terms[i] = x < 0.0 ? x : 0.0;
  }
}

__global__ void k_dual_combine(int nchunks_node, int nchunks_edge, int b, const double* __restrict__ parts,
                               double* __restrict__ out) {
  // combine_partials (parallel.cpp:102-106) in chunk order; b*node + edge (dual.cpp:122)
  double ns = 0.0, es = 0.0;
  for (int i = 0; i < nchunks_node; ++i) ns = dadd(ns, parts[i]);
  for (int i = 0; i < nchunks_edge; ++i) es = dadd(es, parts[nchunks_node + i]);
  *out = dadd(dmul((double)b, ns), es);
}

double dual_objective_device(const f2m_graph& g, const double* d_lam_pos, int b, double* h_async) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int nn = (int)((t.n + kNodeChunk - 1) / kNodeChunk);
  const int ne = (int)((t.m + kEdgeChunk - 1) / kEdgeChunk);
  DBuf<double> parts(nn + ne + 1, s);
  if (nn + ne > 0) {
    // the reference's per-chunk sequential sums (parallel.cpp chunking), bit-exact (seqsum.cu)
    DBuf<double> terms((size_t)t.n + t.m, s);
    k_dual_terms<<<grid_for((int64_t)t.n + t.m, 256), 256, 0, s>>>(t.n, t.m, t.perm.get(), t.eu.get(), t.ev.get(),
                                                                  g.cost.get(), d_lam_pos, terms.get());
    launched("dual_terms");
    if (t.n > 0) seq_sums_device(terms.get(), t.n, kNodeChunk, parts.get(), s);
    if (t.m > 0) seq_sums_device(terms.get() + t.n, t.m, kEdgeChunk, parts.get() + nn, s);
  }
  k_dual_combine<<<1, 1, 0, s>>>(nn, ne, b, parts.get(), parts.get() + nn + ne);
  launched("dual_combine");
  if (h_async) {
    F2M_CUDA(cudaMemcpyAsync(h_async, parts.get() + nn + ne, sizeof(double), cudaMemcpyDeviceToHost, s));
    return NAN;
  }
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
  if (c.num_gpus < 0 || c.num_gpus > 32) throw Error(F2M_E_ARGUMENT, "EngineConfig: num_gpus must be in [0, 32]");
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
                        DBuf<double>& d_lam_out, f2m_convergence_report& rep, double* h_dual_async) {
  validate_engine(cfg);
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const auto t0 = std::chrono::steady_clock::now();
  DBuf<double> l0(std::max(t.n, 1), s), l1(std::max(t.n, 1), s);
  int* init_err = nullptr;
  if (d_init) {
    if (t.n > 0)
      F2M_CUDA(cudaMemcpyAsync(l0.get(), d_init, sizeof(double) * t.n, cudaMemcpyDeviceToDevice, s));
  } else {
    // the init's watchdog flag is collected with the sweep's own synchronisation
    init_err = reinterpret_cast<int*>(pinned_scratch() + 20);
    *init_err = 0;
    initial_state_device(g, cfg, l0.get(), init_err);
  }
  // threshold = eps * mean_cost (dual.cpp:221); with the mean still unknown the v5 kernel
  // computes it during the solve
  const bool defer = !g.mean_known && cfg.mode == 0 && cfg.max_sweeps > 0;
  const double threshold = defer ? 0.0 : cfg.eps * graph_mean(g);
  rep.converged = 0;
  rep.sweeps = 0;
  rep.final_max_abs_delta = INFINITY;
  DBuf<double>* result = &l0;
  // EngineConfig::num_gpus: the Jacobi sweeps on several GPUs (multi.cu), clamped to the slices
  const int64_t nsl = ((int64_t)t.n + 31) / 32;
  const int world = (int)std::max<int64_t>(1, std::min<int64_t>(cfg.num_gpus, nsl));
  if (cfg.max_sweeps > 0) {
    check_degree(g, cfg.b);
    if (cfg.mode == 0 && world > 1 && !g.allpairs) {
      if (init_err) {  // lambda_0 (l0) goes to the replicas: collect the init's watchdog flag first
        F2M_CUDA(cudaStreamSynchronize(s));
        if (*init_err) throw Error(F2M_E_TIMEOUT, "initial-state kernel: dependency wait watchdog fired");
      }
      solve_duals_multi(g, cfg, world, l0.get(), l1, rep);
      F2M_CUDA(cudaSetDevice(t.dev));
      result = &l1;
    } else if (cfg.mode == 0) {
      SweepResult r = run_jacobi(g, cfg, l0.get(), l1.get(), cfg.max_sweeps, threshold, nullptr,
                                 defer ? cfg.eps : 0.0);
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
  rep.dual_value = dual_objective_device(g, result->get(), cfg.b, h_dual_async);
  if (init_err) {  // collected by the sweep's (or, without sweeps, this) synchronisation
    if (cfg.max_sweeps <= 0 || cfg.mode != 0) F2M_CUDA(cudaStreamSynchronize(s));
    if (*init_err) throw Error(F2M_E_TIMEOUT, "initial-state kernel: dependency wait watchdog fired");
  }
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

extern "C" int f2m_jacobi_deltas(const f2m_graph* g, const f2m_engine_config* cfg, const double* lambda,
                                 double* delta) {
  return guard([&] {
    validate_engine(*cfg);
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.n == 0) return;
    check_degree(*g, cfg->b);
    cudaStream_t s = t.stream;
    DBuf<double> l0(t.n, s), d0(t.n, s);
    upload_lambda(*g, lambda, l0.get());
    const unsigned blocks = grid_for((int64_t)t.n * 32, 256);
    switch (cfg->b) {
#define F2M_AD(BB) case BB: k_all_deltas<BB><<<blocks, 256, 0, s>>>(t.n, t.deg.get(), t.sptr.get(), t.scol.get(), g->scost.get(), l0.get(), cfg->update, d0.get()); break;
      F2M_AD(1) F2M_AD(2) F2M_AD(3) F2M_AD(4) F2M_AD(5) F2M_AD(6) F2M_AD(7) F2M_AD(8)
#undef F2M_AD
    }
    launched("all_deltas");
    download_lambda(*g, d0.get(), delta);
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

namespace f2mgpu {
void note_sweep_kernel(double ms, int sweeps) {
  g_last_sweep_ms = ms;
  g_last_sweep_count = sweeps;
}
}  // namespace f2mgpu

extern "C" const char* f2m_last_sweep_kernel_desc(void) { return g_last_sweep_desc.c_str(); }

extern "C" int f2m_set_allpairs_mode(int mode) {
  return guard([&] {
    if (mode < 0 || mode > 2) throw Error(F2M_E_ARGUMENT, "f2m_set_allpairs_mode: mode must be 0, 1 or 2");
    g_allpairs_mode.store(mode);
  });
}

// debug builds only (-DF2M_WARP_PROFILE): the per-warp cycle accounting of the last sweep launch,
// [160 CTAs][32 warps][8] = {halo wait, boundary rows, interior rows, end barrier, sweeps,
// interior slices, interior slot columns, boundary slice width}
extern "C" int f2m_debug_warp_profile(unsigned long long* out, size_t count) {
  return guard([&] {
#ifdef F2M_WARP_PROFILE
    if (count < (size_t)kProfCtas * kProfWarps * kProfFields) throw Error(F2M_E_ARGUMENT, "warp profile: buffer too small");
    F2M_CUDA(cudaMemcpyFromSymbol(out, g_wprof, sizeof(g_wprof)));
#else
    (void)out;
    (void)count;
    throw Error(F2M_E_ARGUMENT, "warp profile: not a -DF2M_WARP_PROFILE build");
#endif
  });
}

// debug builds only (-DF2M_WARP_PROFILE): per-CTA event clocks of 64 sweeps of the last launch
// (zeroed first when `reset`), [160 CTAs][64 sweeps][4] = {sweep start, last boundary row
// published, halo staged, end-of-sweep barrier} (tools/sweep_trace.py)
extern "C" int f2m_debug_sweep_trace(unsigned long long* out, size_t count, int reset) {
  return guard([&] {
#ifdef F2M_WARP_PROFILE
    if (reset) {
      static unsigned long long zero[kProfCtas][kTraceN][4];
      F2M_CUDA(cudaMemcpyToSymbol(g_strace, zero, sizeof(zero)));
      return;
    }
    if (count < (size_t)kProfCtas * kTraceN * 4) throw Error(F2M_E_ARGUMENT, "sweep trace: buffer too small");
    F2M_CUDA(cudaMemcpyFromSymbol(out, g_strace, sizeof(g_strace)));
#else
    (void)out;
    (void)count;
    (void)reset;
    throw Error(F2M_E_ARGUMENT, "sweep trace: not a -DF2M_WARP_PROFILE build");
#endif
  });
}

extern "C" int f2m_last_sweep_kernel_ms(double* ms, int* sweeps) {
  if (ms) *ms = g_last_sweep_ms;
  if (sweeps) *sweeps = g_last_sweep_count;
  return F2M_OK;
}


// ---------------------------------------------------------------- multi-GPU persistent sweep
// The partition-resident sweep kernel spread over `world` ranks: the graph (identical on every
// rank) is partitioned into g_total = world x Gp CTAs (f2m_set_sweep_partition before building
// it); rank r launches CTAs [r*Gp, (r+1)*Gp) plus its own master. LL and max rings are stored
// into every rank's copy (peer memory), so every master issues the same verdicts.
extern "C" int f2m_sweep_multi_info(const f2m_graph* g, int rank, int world, int* g_total, int* resident,
                                    int64_t* ll_words, int64_t* cmax_words, int* begin, int* end) {
  return f2mgpu::guard([&] {
    using namespace f2mgpu;
    const Topology& t = *g->topo;
    if (!t.v2) throw Error(F2M_E_ARGUMENT, "multi sweep: the graph has no partition-resident layout");
    if (world < 1 || t.sweep_ctas % world) throw Error(F2M_E_ARGUMENT, "multi sweep: partition not divisible by world");
    if (rank < 0 || rank >= world) throw Error(F2M_E_INDEX, "multi sweep: rank outside [0, world)");
    const int G = t.sweep_ctas, Gp = G / world;
    *g_total = G;
    *resident = t.resident ? 1 : 0;
    *ll_words = (int64_t)kLLRing * std::max(t.nboundary, 1) * 2;
    *cmax_words = (int64_t)kCmaxRing * G * 2;
    int32_t lo[2];
    F2M_CUDA(cudaMemcpy(&lo[0], t.cta_lo.get() + rank * Gp, sizeof(int32_t), cudaMemcpyDeviceToHost));
    F2M_CUDA(cudaMemcpy(&lo[1], t.cta_lo.get() + (rank + 1) * Gp, sizeof(int32_t), cudaMemcpyDeviceToHost));
    *begin = std::min(lo[0] * 32, t.n);
    *end = std::min(lo[1] * 32, t.n);
  });
}

extern "C" size_t f2m_sweep_multi_ctl_bytes(void) { return sizeof(f2mgpu::Sweep4Ctl); }

namespace f2mgpu {
// bit r of mask[i]: a CTA of rank r has LL entry i (a boundary node of another CTA) in its halo
__global__ void k_ll_mask(int G, int gp, const int32_t* __restrict__ halo_off, const int32_t* __restrict__ halo_pub,
                          uint32_t* __restrict__ mask) {
  const int c = blockIdx.x;
  if (c >= G) return;
  const uint32_t bit = 1u << (c / gp);
  for (int h = halo_off[c] + threadIdx.x; h < halo_off[c + 1]; h += blockDim.x) atomicOr(&mask[halo_pub[h]], bit);
}
}  // namespace f2mgpu

namespace f2mgpu {
// per-sweep remote LL stores of rank r: every boundary node of r's CTAs is stored into each OTHER
// rank whose CTAs read it (popcount of its rank mask without bit r)
__global__ void k_ll_remote(int G, int gp, int rank, const int32_t* __restrict__ boff,
                            const uint32_t* __restrict__ mask, unsigned long long* __restrict__ count) {
  const int lo = boff[rank * gp], hi = boff[min(G, (rank + 1) * gp)];
  unsigned long long local = 0;
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
    local += __popc(mask[i] & ~(1u << rank));
  if (local) atomicAdd(count, local);
}
}  // namespace f2mgpu

extern "C" int f2m_sweep_multi_traffic(const f2m_graph* g, int rank, int world, int64_t* remote_ll_stores,
                                       int64_t* remote_max_stores) {
  return f2mgpu::guard([&] {
    using namespace f2mgpu;
    const Topology& t = *g->topo;
    if (world < 1 || !t.v2 || t.sweep_ctas % world) throw Error(F2M_E_ARGUMENT, "multi sweep: bad partition");
    if (rank < 0 || rank >= world) throw Error(F2M_E_INDEX, "multi sweep: rank outside [0, world)");
    if (world > 32) throw Error(F2M_E_ARGUMENT, "multi sweep: at most 32 ranks");
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    const int G = t.sweep_ctas, Gp = G / world;
    const int nb = std::max(t.nboundary, 1);
    DBuf<uint32_t> mask((size_t)nb, s);
    DBuf<unsigned long long> cnt(1, s);
    F2M_CUDA(cudaMemsetAsync(mask.get(), 0, mask.bytes(), s));
    F2M_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
    if (G > 0) {
      k_ll_mask<<<G, 128, 0, s>>>(G, Gp, t.halo_off.get(), t.halo_pub.get(), mask.get());
      launched("ll_mask");
      k_ll_remote<<<64, 256, 0, s>>>(G, Gp, rank, t.boff.get(), mask.get(), cnt.get());
      launched("ll_remote");
    }
    unsigned long long h = 0;
    F2M_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    *remote_ll_stores = (int64_t)h;
    *remote_max_stores = (int64_t)Gp * (world - 1);
  });
}

extern "C" int f2m_sweep_multi_launch(const f2m_graph* g, const f2m_engine_config* cfg, int rank, int world,
                                      double* d_ring, unsigned long long* d_ll,
                                      unsigned long long* const* d_ll_peers, unsigned long long* d_cmax,
                                      unsigned long long* const* d_cmax_peers, double threshold, int max_sweeps,
                                      void* d_ctl, void* stream) {
  return f2mgpu::guard([&] {
    using namespace f2mgpu;
    validate_engine(*cfg);
    const Topology& t = *g->topo;
    if (world < 1 || !t.v2 || t.sweep_ctas % world) throw Error(F2M_E_ARGUMENT, "multi sweep: bad partition");
    if (rank < 0 || rank >= world) throw Error(F2M_E_INDEX, "multi sweep: rank outside [0, world)");
    if (t.n > 0 && t.min_deg <= cfg->b)
      throw Error(F2M_E_DEGREE, "node has degree " + std::to_string(t.min_deg) + " <= b = " + std::to_string(cfg->b));
    const int G = t.sweep_ctas, Gp = G / world;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Sweep4Ctl* ctl = static_cast<Sweep4Ctl*>(d_ctl);
    F2M_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Sweep4Ctl), s));
    Sweep4Args a{};
    a.n = t.n;
    a.sptr = t.sptr.get();
    a.swidth = t.swidth.get();
    a.cta_lo = t.cta_lo.get();
    a.cta_int_hi = t.cta_int_hi.get();
    a.cta_nint = t.cta_nint.get();
    a.boff = t.boff.get();
    a.slidx = t.slidx.get();
    a.scost = g->scost.get();
    a.halo_off = t.halo_off.get();
    a.halo = t.halo.get();
    a.halo_pub = t.halo_pub.get();
    a.gl = d_ring;  // kLamBufs x n; buffer 0 holds lambda_0 (full vector) on entry
    a.gstride = (size_t)std::max(t.n, 1);
    a.ll = d_ll;
    a.nb = std::max(t.nboundary, 1);
    a.sdest = t.sdest.get();
    a.poll_ns = kPollNs;
    a.runahead = 1;
    a.defer_eps = 0.0;
    a.cost = g->cost.get();
    a.m = t.m;
    a.approx_sum = g->approx_sum.get();
    a.mean_out = nullptr;
    a.pair_rows = t.n <= kPairRowsPerCta * G ? 1 : 0;
    a.cmax = d_cmax;
    a.eta = cfg->eta;
    a.update = cfg->update;
    a.threshold = threshold;
    a.max_sweeps = max_sweeps;
    a.record = nullptr;
    a.lam_stride = (int)((((size_t)t.max_local * sizeof(double) + 15) & ~size_t(15)) / sizeof(double));
    a.lam_ring = t.resident ? t.lam_ring : 2;
    a.row_skip = t.resident ? t.row_skip : 0;
    a.halo_stride = (t.max_halo + 3) & ~3;
    a.lid4_stride = (int)t.max_cta_lid4;
    a.cta_base = rank * Gp;
    a.g_total = G;
    a.npeers = world;
    a.ll_peers = d_ll_peers;
    a.cmax_peers = d_cmax_peers;
    if (world > 32) throw Error(F2M_E_ARGUMENT, "multi sweep: at most 32 ranks");
    DBuf<uint32_t> mask((size_t)a.nb, s);
    F2M_CUDA(cudaMemsetAsync(mask.get(), 0, mask.bytes(), s));
    if (G > 0) {
      k_ll_mask<<<G, 128, 0, s>>>(G, Gp, t.halo_off.get(), t.halo_pub.get(), mask.get());
      launched("ll_mask");
    }
    a.ll_mask = mask.get();  // freed (stream-ordered) after the sweep kernel
    g_last_sweep_desc = "k_gdp_sweep5<b=" + std::to_string(cfg->b) +
                        (t.resident ? ", resident, " + std::to_string(kResidentThreads)
                                    : ", streaming, " + std::to_string(kStreamingThreads)) +
                        "> multi-rank (rank " + std::to_string(rank) + "/" + std::to_string(world) + ": " +
                        std::to_string(Gp) + " of " + std::to_string(G) + " partition CTAs + 1 master, LL rings in every rank's memory)";
    dispatch_sweep5(t, cfg->b, a, ctl, Gp + 1, s);
    launched("gdp_sweep5_multi");
  });
}

extern "C" int f2m_sweep_multi_result(const void* d_ctl, int* sweeps, int* converged, double* final_max,
                                      int* out_buffer) {
  return f2mgpu::guard([&] {
    f2mgpu::Sweep4Ctl h;
    F2M_CUDA(cudaMemcpy(&h, d_ctl, sizeof(h), cudaMemcpyDeviceToHost));
    if (h.abort) throw f2mgpu::Error(F2M_E_TIMEOUT, "multi sweep: synchronisation watchdog fired");
    *sweeps = h.sweeps;
    *converged = h.converged;
    *final_max = h.final_max;
    *out_buffer = h.out_buffer;
  });
}

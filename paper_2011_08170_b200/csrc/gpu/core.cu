// core.cu — device/graph plumbing of libf2m_gpu.so: errors, graph creation
// (Graph::from_edges graph.cpp:14-51, with_costs :53-65, jittered solve.cpp:39-47),
// the SELL-32 sweep layout, mean cost, validate_graph (graph.cpp:242-277).
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>

#include <vector>

#include "internal.cuh"

namespace f2mgpu {

std::atomic<uint64_t> g_launches{0};

static thread_local std::string t_last_error;
static thread_local int t_device = 0;

void set_last_error(const std::string& msg) { t_last_error = msg; }

int current_device() { return t_device; }

const cudaDeviceProp& device_props(int dev) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<cudaDeviceProp>> cache(64);
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) throw Error(F2M_E_ARGUMENT, "device index out of range");
  if (!cache[dev]) {
    auto p = std::make_unique<cudaDeviceProp>();
    F2M_CUDA(cudaGetDeviceProperties(p.get(), dev));
    cache[dev] = std::move(p);
    // Scratch buffers are stream-ordered allocations (DBuf). Keep freed memory in the device's
    // pool instead of returning it to the driver at every synchronisation (the default release
    // threshold is 0), so repeated solves do not pay cudaMalloc-class latencies.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return *cache[dev];
}

Topology::~Topology() {
  if (stream) {
    cudaSetDevice(dev);
    eu.release(); ev.release(); perm.release(); iperm.release(); perm0.release(); iperm0.release(); deg.release();
    sptr.release(); swidth.release(); scol.release(); seid.release(); cta_lo.release();
    halo_off.release(); halo.release(); slidx.release();
    cta_int_hi.release(); cta_nint.release(); boff.release(); halo_pub.release();
    sdest.release(); row_nhalo.release();
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

std::shared_ptr<Topology> make_topology(int n, int dev) {
  (void)device_props(dev);  // first use of the device configures its memory pool
  auto t = std::make_shared<Topology>();
  t->dev = dev;
  t->n = n;
  F2M_CUDA(cudaSetDevice(dev));
  F2M_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
  return t;
}

// ---------------------------------------------------------------- kernels

// partition CTA count for graphs built from now on (0: one per SM but one); the multi-GPU sweep
// partitions a replicated graph into world x (SMs - 1) CTAs
int g_sweep_partition = 0;

int64_t* pinned_scratch() {
  thread_local int64_t* p = nullptr;
  // portable: the same thread may drive several devices (f2m_set_device)
  if (!p) F2M_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), 64 * sizeof(int64_t), cudaHostAllocPortable));
  return p;
}

__global__ void k_drop_sentinel(const int64_t* __restrict__ nsel, const uint64_t* __restrict__ keys,
                                uint64_t sentinel, int64_t* __restrict__ out) {
  const int64_t h = *nsel;
  *out = (h > 0 && keys[h - 1] == sentinel) ? h - 1 : h;  // drop the "not halo" sentinel
}

__global__ void k_edge_keys(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            uint64_t* __restrict__ keys, int64_t* __restrict__ idx) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint32_t a = (uint32_t)min(u[e], v[e]), b = (uint32_t)max(u[e], v[e]);
  keys[e] = ((uint64_t)a << 32) | b;
  idx[e] = e;
}

__global__ void k_unpack_edges(int64_t m, const uint64_t* __restrict__ keys,
                               const int64_t* __restrict__ idx, const double* __restrict__ cin,
                               int32_t* __restrict__ u, int32_t* __restrict__ v,
                               double* __restrict__ cout) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  u[e] = (int32_t)(keys[e] >> 32);
  v[e] = (int32_t)(keys[e] & 0xffffffffu);
  cout[e] = cin[idx[e]];
}

__global__ void k_iota(int n, int32_t* __restrict__ a, int32_t* __restrict__ b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { a[i] = i; b[i] = i; }
}

// Degree by position: self-loops count once (graph.cpp:30-31).
__global__ void k_degrees(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                          const int32_t* __restrict__ perm, int32_t* __restrict__ deg) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  atomicAdd(&deg[perm[eu[e]]], 1);
  if (ev[e] != eu[e]) atomicAdd(&deg[perm[ev[e]]], 1);
}

// Slice widths (max degree over the 32 positions of a slice) and slice sizes.
__global__ void k_slice_width(int n, int64_t nslices, const int32_t* __restrict__ deg,
                              int32_t* __restrict__ width, int64_t* __restrict__ size) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int w = 0;
  const int64_t p0 = s * 32;
  for (int l = 0; l < 32; ++l) {
    const int64_t p = p0 + l;
    if (p < n) w = max(w, deg[p]);
  }
  width[s] = w;
  size[s] = (int64_t)w * 32;
}

__global__ void k_fill_pad(int64_t nslices, const int64_t* __restrict__ sptr,
                           int32_t* __restrict__ scol, int32_t* __restrict__ seid) {
  // one warp per slice: padding col = own position, eid = -1
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  for (int64_t t = sptr[s] + lane; t < sptr[s + 1]; t += 32) {
    scol[t] = (int32_t)(s * 32 + lane);
    seid[t] = -1;
  }
}

__global__ void k_fill_sell(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                            const int32_t* __restrict__ perm, const int64_t* __restrict__ sptr,
                            int32_t* __restrict__ fill, int32_t* __restrict__ scol,
                            int32_t* __restrict__ seid) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int pu = perm[eu[e]], pv = perm[ev[e]];
  {
    const int j = atomicAdd(&fill[pu], 1);
    const int64_t t = sptr[pu >> 5] + (int64_t)j * 32 + (pu & 31);
    scol[t] = pv;
    seid[t] = (int32_t)e;
  }
  if (pu != pv) {
    const int j = atomicAdd(&fill[pv], 1);
    const int64_t t = sptr[pv >> 5] + (int64_t)j * 32 + (pv & 31);
    scol[t] = pu;
    seid[t] = (int32_t)e;
  }
}

// CTA partition of slices balanced by padded slot count: cta_lo[c] = first slice whose
// start offset is >= c * total / ctas.
__global__ void k_partition(int ctas, int64_t nslices, const int64_t* __restrict__ sptr,
                            int32_t* __restrict__ lo) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > ctas) return;
  if (c == ctas) { lo[c] = (int32_t)nslices; return; }
  const int64_t total = sptr[nslices];
  // target in slots, mixed with a per-slice fixed cost so empty-ish slices still spread
  const double target = (double)c / ctas;
  int64_t a = 0, b = nslices;
  while (a < b) {
    const int64_t mid = (a + b) / 2;
    const double f = ((double)sptr[mid] + 64.0 * mid) / ((double)total + 64.0 * nslices);
    if (f < target) a = mid + 1; else b = mid;
  }
  lo[c] = (int32_t)a;
}

__global__ void k_scost(int64_t slots, const int32_t* __restrict__ seid,
                        const double* __restrict__ cost, double* __restrict__ scost) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= slots) return;
  const int32_t e = seid[t];
  scost[t] = e >= 0 ? cost[e] : CUDART_INF;
}


__global__ void k_jitter(int64_t m, const double* __restrict__ cin, double amplitude,
                         uint64_t state0, double* __restrict__ cout) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  // graph.edge(e).cost + amplitude * rng.next_double()  (solve.cpp:44), no contraction
  cout[e] = dadd(cin[e], dmul(amplitude, splitmix64_double_at(state0, (uint64_t)e)));
}

// validate_graph edge checks (graph.cpp:245-263): first offending edge in edge order.
__global__ void k_validate(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                           const double* __restrict__ cost, unsigned long long* __restrict__ first) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  int kind = 0;
  if (eu[e] == ev[e]) kind = 1;                                        // self-loop
  else if (e > 0 && eu[e - 1] == eu[e] && ev[e - 1] == ev[e]) kind = 2; // duplicate
  else if (!(cost[e] >= 0.0)) kind = 3;                                // negative cost
  if (kind) atomicMin(first, ((unsigned long long)e << 2) | (unsigned long long)kind);
}

__global__ void k_minmax_deg(int n, const int32_t* __restrict__ deg, int* __restrict__ mn,
                             int* __restrict__ mx) {
  int lo = INT_MAX, hi = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    lo = min(lo, deg[i]);
    hi = max(hi, deg[i]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mn, lo);
    atomicMax(mx, hi);
  }
}

__global__ void k_gather_i32(int n, const int32_t* __restrict__ src, const int32_t* __restrict__ idx,
                             int32_t* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_gather_f64(int n, const double* __restrict__ src, const int32_t* __restrict__ idx,
                             double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_scatter_f64(int n, const double* __restrict__ src, const int32_t* __restrict__ idx,
                              double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

__global__ void k_incidence_keys(int64_t m, const int32_t* __restrict__ eu,
                                 const int32_t* __restrict__ ev, const int64_t* __restrict__ off,
                                 int32_t* __restrict__ cur, int32_t* __restrict__ ids) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  ids[off[eu[e]] + atomicAdd(&cur[eu[e]], 1)] = (int32_t)e;
  if (ev[e] != eu[e]) ids[off[ev[e]] + atomicAdd(&cur[ev[e]], 1)] = (int32_t)e;
}


// ---- permutation application: position i takes the node previously at old_of_new[i]
__global__ void k_window_apply(int n, const int32_t* __restrict__ old_of_new, const int32_t* __restrict__ deg_old,
                               const int32_t* __restrict__ iperm_old, int32_t* __restrict__ deg_new,
                               int32_t* __restrict__ iperm_new, int32_t* __restrict__ perm_new) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int o = old_of_new[i];
  deg_new[i] = deg_old[o];
  const int orig = iperm_old[o];
  iperm_new[i] = orig;
  perm_new[orig] = i;
}


// ---- CTA partition and CTA-local node order (persistent sweep kernel)
__global__ void k_slice_weight(int n, int64_t nslices, const int32_t* __restrict__ deg, int64_t* __restrict__ w) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int64_t acc = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t p = s * 32 + l;
    if (p < n) acc += deg[p];
  }
  w[s] = acc;
}

__global__ void k_boundary(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                           const int32_t* __restrict__ perm, const int32_t* __restrict__ cos,
                           uint8_t* __restrict__ bnd) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int pu = perm[eu[e]], pv = perm[ev[e]];
  if (cos[pu >> 5] != cos[pv >> 5]) {
    bnd[pu] = 1;
    bnd[pv] = 1;
  }
}

__global__ void k_local_keys(int n, const int32_t* __restrict__ deg, const uint8_t* __restrict__ bnd,
                             const int32_t* __restrict__ cos, int dbits, int max_deg,
                             uint64_t* __restrict__ key, int32_t* __restrict__ val, int32_t* __restrict__ nint) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int c = cos[p >> 5];
  // CTA (keeps the partition), interior before boundary, then degree descending (capped at
  // max_deg: the local order only shapes the SELL padding, results do not depend on it), packed
  // into bits(G) + 1 + dbits bits so the (stable) radix sort runs only the passes it needs
  key[p] = ((uint64_t)(uint32_t)c << (dbits + 1)) | ((uint64_t)bnd[p] << dbits) |
           (uint32_t)(max_deg - min(deg[p], max_deg));
  val[p] = p;
  // a warp's 32 positions are one slice, hence one CTA: one atomic per warp, not per node (147
  // contended counters cost ~27 us at 100k)
  const unsigned interior = __ballot_sync(__activemask(), !bnd[p]);
  if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && interior) atomicAdd(&nint[c], __popc(interior));
}

__global__ void k_int_hi(int ctas, const int32_t* __restrict__ lo, const int32_t* __restrict__ nint,
                         int32_t* __restrict__ int_hi) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ctas) int_hi[c] = lo[c] + nint[c] / 32;  // whole slices of interior nodes
}

// ---- v2 local index space
__global__ void k_cta_of_slice(int ctas, const int32_t* __restrict__ lo, int32_t* __restrict__ cos) {
  const int c = blockIdx.x;
  for (int s = lo[c] + threadIdx.x; s < lo[c + 1]; s += blockDim.x) cos[s] = c;
}

__device__ __forceinline__ void own_range(int c, int n, const int32_t* __restrict__ lo, int& p0, int& p1) {
  p0 = lo[c] * 32;
  p1 = min(lo[c + 1] * 32, n);
  if (p1 < p0) p1 = p0;
}

// one warp per slice: halo key (cta << 32 | q) for every neighbour q outside the owner's range
__global__ void k_halo_keys(int n, int64_t nslices, const int64_t* __restrict__ sptr,
                            const int32_t* __restrict__ scol, const int32_t* __restrict__ seid,
                            const int32_t* __restrict__ cos, const int32_t* __restrict__ lo, int qbits,
                            uint64_t sentinel, uint64_t* __restrict__ keys) {
  // key = (CTA << qbits) | position, packed so the radix sort runs only the passes it needs;
  // non-halo slots get the sentinel (all ones: larger than every real key), sorted last
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int c = cos[s];
  int p0, p1;
  own_range(c, n, lo, p0, p1);
  for (int64_t t = sptr[s] + lane; t < sptr[s + 1]; t += 32) {
    const int q = scol[t];
    const bool halo = seid[t] >= 0 && (q < p0 || q >= p1);
    keys[t] = halo ? (((uint64_t)(uint32_t)c << qbits) | (uint32_t)q) : sentinel;
  }
}

__global__ void k_halo_split(int64_t h, const uint64_t* __restrict__ keys, int qbits, int32_t* __restrict__ halo,
                             int32_t* __restrict__ cnt, const int64_t* __restrict__ dh = nullptr) {
  // dh: the entry count on the device (the grid covers an upper bound h, no host round trip)
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= h || (dh && i >= *dh)) return;
  halo[i] = (int32_t)(keys[i] & ((1ull << qbits) - 1));
  // keys are sorted by CTA: lanes with the same CTA add once (a handful of contended counters)
  const int c = (int)(keys[i] >> qbits);
  const unsigned same = __match_any_sync(__activemask(), c);
  if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&cnt[c], __popc(same));
}

__global__ void k_local_sizes(int ctas, int n, const int32_t* __restrict__ lo, const int32_t* __restrict__ hoff,
                              const int64_t* __restrict__ sptr, const int32_t* __restrict__ swidth,
                              int* __restrict__ max_local, unsigned long long* __restrict__ max_slots) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ctas) return;
  int p0, p1;
  own_range(c, n, lo, p0, p1);
  atomicMax(max_local, (p1 - p0) + (hoff[c + 1] - hoff[c]));
  atomicMax(max_local + 1, hoff[c + 1] - hoff[c]);  // halo entries alone
  atomicMax(max_local + 2, lo[c + 1] - lo[c]);      // slices
  atomicMax(max_slots, (unsigned long long)(sptr[lo[c + 1]] - sptr[lo[c]]));
  unsigned long long l4 = 0;  // packed local-index entries (ushort4, widths padded to 4)
  for (int i = lo[c]; i < lo[c + 1]; ++i) l4 += 32ull * (unsigned)((swidth[i] + 3) / 4);
  atomicMax(max_slots + 1, l4);
}

__global__ void k_slot_lidx(int n, int64_t nslices, const int64_t* __restrict__ sptr,
                            const int32_t* __restrict__ scol, const int32_t* __restrict__ seid,
                            const int32_t* __restrict__ cos, const int32_t* __restrict__ lo,
                            const int32_t* __restrict__ hoff, const int32_t* __restrict__ halo,
                            uint16_t* __restrict__ slidx) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int c = cos[s];
  int p0, p1;
  own_range(c, n, lo, p0, p1);
  const int own = p1 - p0;
  const int h0 = hoff[c], h1 = hoff[c + 1];
  const int p = (int)(s * 32 + lane);
  for (int64_t t = sptr[s] + lane; t < sptr[s + 1]; t += 32) {
    int li;
    if (seid[t] < 0) {
      li = min(max(p - p0, 0), max(own - 1, 0));  // padding: own slot, cost +inf
    } else {
      const int q = scol[t];
      if (q >= p0 && q < p1) {
        li = q - p0;
      } else {
        int a = h0, b = h1;
        while (a < b) { const int mid = (a + b) >> 1; if (halo[mid] < q) a = mid + 1; else b = mid; }
        li = own + (a - h0);
      }
    }
    slidx[t] = (uint16_t)li;
  }
}

// halo-last slot order per row (stable within each class) + halo slot count per row
__global__ void k_halo_last(int n, int64_t nslices, const int64_t* __restrict__ sptr,
                            const int32_t* __restrict__ swidth, const uint16_t* __restrict__ slidx,
                            const int32_t* __restrict__ cos, const int32_t* __restrict__ lo,
                            int32_t* __restrict__ sdest, uint8_t* __restrict__ nhalo) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  int p0, p1;
  own_range(cos[s], n, lo, p0, p1);
  const int own = p1 - p0;
  const int w = swidth[s];
  const int64_t base = sptr[s] + lane;
  int nh = 0;
  for (int j = 0; j < w; ++j) nh += slidx[base + 32 * (int64_t)j] >= own;
  int io = 0, ih = w - nh;
  for (int j = 0; j < w; ++j) {
    const bool h = slidx[base + 32 * (int64_t)j] >= own;
    sdest[base + 32 * (int64_t)j] = (int32_t)(base + 32 * (int64_t)(h ? ih++ : io++));
  }
  const int64_t p = s * 32 + lane;
  if (p < n) nhalo[p] = (uint8_t)min(nh, 255);
}

// ---- LL exchange: boundary publication indices
__global__ void k_boundary_counts(int ctas, int n, const int32_t* __restrict__ lo, const int32_t* __restrict__ nint,
                                  int32_t* __restrict__ cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > ctas) return;
  if (c == ctas) { cnt[c] = 0; return; }
  int p0, p1;
  own_range(c, n, lo, p0, p1);
  cnt[c] = max(0, (p1 - p0) - nint[c]);
}

__global__ void k_halo_pub(int64_t h, const int32_t* __restrict__ halo, const int32_t* __restrict__ cos,
                           const int32_t* __restrict__ lo, const int32_t* __restrict__ nint,
                           const int32_t* __restrict__ boff, int32_t* __restrict__ pub) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= h) return;
  const int q = halo[i];
  const int c = cos[q >> 5];
  pub[i] = boff[c] + (q - lo[c] * 32 - nint[c]);  // q is a boundary node of its owner (symmetric graph)
}

// ---------------------------------------------------------------- host helpers

void sort_edges(Topology& t, DBuf<int32_t>& eu, DBuf<int32_t>& ev, DBuf<double>& cost) {
  const int64_t m = t.m;
  cudaStream_t s = t.stream;
  DBuf<uint64_t> k0(m, s), k1(m, s);
  DBuf<int64_t> i0(m, s), i1(m, s);
  if (m > 0) {
    k_edge_keys<<<grid_for(m, 256), 256, 0, s>>>(m, eu.get(), ev.get(), k0.get(), i0.get());
    launched("edge_keys");
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.get(), k1.get(), i0.get(), i1.get(),
                                             m, 0, 64, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, k0.get(), k1.get(), i0.get(), i1.get(),
                                             m, 0, 64, s));
    launched("radix_sort_edges");
  }
  t.eu.alloc(m, s);
  t.ev.alloc(m, s);
  DBuf<double> c2(m, s);
  if (m > 0) {
    k_unpack_edges<<<grid_for(m, 256), 256, 0, s>>>(m, k1.get(), i1.get(), cost.get(), t.eu.get(),
                                                   t.ev.get(), c2.get());
    launched("unpack_edges");
  }
  cost = std::move(c2);
}

void identity_perm(Topology& t) {
  t.perm.alloc(t.n, t.stream);
  t.iperm.alloc(t.n, t.stream);
  if (t.n > 0) {
    k_iota<<<grid_for(t.n, 256), 256, 0, t.stream>>>(t.n, t.perm.get(), t.iperm.get());
    launched("iota");
  }
}

// v2 sweep structures: halo lists, per-slot local indices, CTA adjacency, smem plan.
static void build_local_index(Topology& t) {
  cudaStream_t s = t.stream;
  const int n = t.n, G = t.sweep_ctas;
  t.v2 = false;
  t.resident = false;
  if (n == 0 || t.nslices == 0) return;
  DBuf<int32_t> cos(t.nslices, s);
  k_cta_of_slice<<<G, 128, 0, s>>>(G, t.cta_lo.get(), cos.get());
  launched("cta_of_slice");
  const int64_t slots = t.sell_slots;
  // halo entries
  const int qbits = std::max(bit_width(n - 1), 1);
  const int key_bits = bit_width(G) + qbits;  // 2^bit_width(G) > G - 1: the all-ones sentinel is unused
  const uint64_t sentinel = (key_bits >= 64) ? ~0ULL : ((1ull << key_bits) - 1);
  DBuf<uint64_t> k0(std::max<int64_t>(slots, 1), s), k1(std::max<int64_t>(slots, 1), s);
  DBuf<int64_t> nsel(1, s), hcnt(1, s);
  F2M_CUDA(cudaMemsetAsync(hcnt.get(), 0, sizeof(int64_t), s));
  int64_t h = 0;
  if (slots > 0) {
    k_halo_keys<<<grid_for(t.nslices * 32, 256), 256, 0, s>>>(n, t.nslices, t.sptr.get(), t.scol.get(),
                                                             t.seid.get(), cos.get(), t.cta_lo.get(), qbits,
                                                             sentinel, k0.get());
    launched("halo_keys");
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0.get(), k1.get(), slots, 0, key_bits, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k0.get(), k1.get(), slots, 0, key_bits, s));
    launched("sort_halo");
    tmp = 0;
    F2M_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, k1.get(), k0.get(), nsel.get(), slots, s));
    DBuf<char> tb2(tmp, s);
    F2M_CUDA(cub::DeviceSelect::Unique(tb2.get(), tmp, k1.get(), k0.get(), nsel.get(), slots, s));
    launched("unique_halo");
    k_drop_sentinel<<<1, 1, 0, s>>>(nsel.get(), k0.get(), sentinel, hcnt.get());
    launched("drop_sentinel");
  }
  // the halo count comes back with the sizes below: until then the halo list is sized (and the
  // split launched) for its bound, the slot count
  t.halo.alloc(std::max<int64_t>(slots, 1), s);
  t.halo_off.alloc(G + 1, s);
  {
    DBuf<int32_t> cnt(G + 1, s);
    F2M_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (G + 1), s));
    if (slots > 0) {
      k_halo_split<<<grid_for(slots, 256), 256, 0, s>>>(slots, k0.get(), qbits, t.halo.get(), cnt.get(), hcnt.get());
      launched("halo_split");
    }
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), t.halo_off.get(), G + 1, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, cnt.get(), t.halo_off.get(), G + 1, s));
    launched("scan_halo");
  }
  // LL publication offsets (boundary nodes of each CTA, in position order)
  t.boff.alloc(G + 1, s);
  {
    DBuf<int32_t> cnt(G + 1, s);
    k_boundary_counts<<<grid_for(G + 1, 128), 128, 0, s>>>(G, n, t.cta_lo.get(), t.cta_nint.get(), cnt.get());
    launched("boundary_counts");
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), t.boff.get(), G + 1, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, cnt.get(), t.boff.get(), G + 1, s));
    launched("scan_boundary");
  }
  // sizes: local index space, halo, slots, slices, packed indices, halo count and boundary count
  // with ONE synchronisation
  int max_slices = 0;
  int64_t max_lid4 = 0;  // resident: packed local indices, 4 slots per 8-byte entry, widths padded to 4
  {
    DBuf<int> ml(3, s);
    DBuf<unsigned long long> ms(2, s);
    F2M_CUDA(cudaMemsetAsync(ml.get(), 0, 3 * sizeof(int), s));
    F2M_CUDA(cudaMemsetAsync(ms.get(), 0, 2 * sizeof(unsigned long long), s));
    k_local_sizes<<<grid_for(G, 128), 128, 0, s>>>(G, n, t.cta_lo.get(), t.halo_off.get(), t.sptr.get(),
                                                   t.swidth.get(), ml.get(), ms.get());
    launched("local_sizes");
    int64_t* hs = pinned_scratch();
    F2M_CUDA(cudaMemcpyAsync(hs + 1, ml.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaMemcpyAsync(hs + 4, ms.get(), 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaMemcpyAsync(hs + 6, hcnt.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaMemcpyAsync(hs + 7, t.boff.get() + G, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    h = hs[6];
    t.max_local = reinterpret_cast<const int*>(hs + 1)[0];
    t.max_halo = reinterpret_cast<const int*>(hs + 1)[1];
    max_slices = reinterpret_cast<const int*>(hs + 1)[2];
    t.max_cta_slots = hs[4];
    max_lid4 = hs[5];
    t.nboundary = reinterpret_cast<const int32_t*>(hs + 7)[0];
  }
  const size_t limit = sweep_smem_limit(t.dev);
  const size_t lam_bytes = (size_t)t.max_local * sizeof(double);
  if (t.max_local > 65535 || lam_bytes > limit) return;  // v1 kernel (global gathers)
  // per-slot local indices
  t.slidx.alloc(std::max<int64_t>(slots, 1), s);
  if (slots > 0) {
    k_slot_lidx<<<grid_for(t.nslices * 32, 256), 256, 0, s>>>(n, t.nslices, t.sptr.get(), t.scol.get(), t.seid.get(),
                                                             cos.get(), t.cta_lo.get(), t.halo_off.get(),
                                                             t.halo.get(), t.slidx.get());
    launched("slot_lidx");
  }
  t.sdest.alloc(std::max<int64_t>(slots, 1), s);
  t.row_nhalo.alloc(std::max(n, 1), s);
  if (slots > 0) {
    k_halo_last<<<grid_for(t.nslices * 32, 256), 256, 0, s>>>(n, t.nslices, t.sptr.get(), t.swidth.get(),
                                                             t.slidx.get(), cos.get(), t.cta_lo.get(),
                                                             t.sdest.get(), t.row_nhalo.get());
    launched("halo_last");
  }
  // LL publication indices of the halo entries
  t.halo_pub.alloc(std::max<int64_t>(h, 1), s);
  {
    if (h > 0) {
      k_halo_pub<<<grid_for(h, 256), 256, 0, s>>>(h, t.halo.get(), cos.get(), t.cta_lo.get(), t.cta_nint.get(),
                                                  t.boff.get(), t.halo_pub.get());
      launched("halo_pub");
    }
  }
  // [lam regions][halo LL ids (max halo ints, 16-byte aligned)][resident: cost + local index per slot]
  const size_t lam_aligned = (lam_bytes + 15) & ~size_t(15);
  const size_t ids_bytes = (((size_t)t.max_halo * sizeof(int)) + 15) & ~size_t(15);
  t.max_cta_lid4 = max_lid4;
  const size_t slice_bytes = 16 + (size_t)max_slices * sizeof(int4);
  size_t resident_bytes = 2 * lam_aligned + ids_bytes + (size_t)t.max_cta_slots * sizeof(double) +
                          (size_t)max_lid4 * 8 + slice_bytes;
  const size_t streaming_bytes = lam_aligned + ids_bytes + slice_bytes;
  if (streaming_bytes > limit) return;  // v1 kernel
  // The sweep kernel keeps per-sweep CTA maxima in a ring of kCmaxRing (64) slots. A CTA starts
  // sweep s+1 only once the master has issued verdict s-7, and the master reads a window of 16
  // sweeps from its next verdict on, so a slot is rewritten (sweep k+64) only long after the master
  // has consumed it (window end <= verdict + 16 < k + 56): the ring is race-free for any G. The
  // grid itself is one CTA per SM (G + master <= SM count); 256 bounds the partition tables.
  if (G > 4096) return;  // v1 kernel
  t.v2 = true;
  t.resident = resident_bytes <= limit;
  // per-row tail budgets (8 bytes per own row, after the slice table) when they fit
  t.row_skip = 0;
  if (t.resident && F2M_ROW_SKIP && resident_bytes + 16 + (size_t)t.max_local * 8 <= limit) {
    t.row_skip = 1;
    resident_bytes += 16 + (size_t)t.max_local * 8;
  }
  t.smem_bytes = t.resident ? resident_bytes : streaming_bytes;
  // eight multiplier regions (the last 8 sweeps) when they fit: no per-sweep global copy of lambda
  t.lam_ring = 2;
  if (t.resident && F2M_LAM_RING8 && resident_bytes + 6 * lam_aligned <= limit) {
    t.lam_ring = 8;
    t.smem_bytes = resident_bytes + 6 * lam_aligned;
  }
}

void finalize_topology(Topology& t) {
  cudaStream_t s = t.stream;
  const int n = t.n;
  const int64_t m = t.m;
  t.deg.alloc(n, s);
  if (n > 0) F2M_CUDA(cudaMemsetAsync(t.deg.get(), 0, sizeof(int32_t) * n, s));
  if (m > 0) {
    k_degrees<<<grid_for(m, 256), 256, 0, s>>>(m, t.eu.get(), t.ev.get(), t.perm.get(), t.deg.get());
    launched("degrees");
  }
  // keep the spatial order itself: a re-partitioned replica (multi.cu) starts from it, not from
  // the CTA-local order below (which is only coherent at this partition's granularity)
  t.perm0.alloc(n, s);
  t.iperm0.alloc(n, s);
  if (n > 0) {
    F2M_CUDA(cudaMemcpyAsync(t.perm0.get(), t.perm.get(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    F2M_CUDA(cudaMemcpyAsync(t.iperm0.get(), t.iperm.get(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  }
  // CTA partition (contiguous slice ranges balanced by degree + a per-slice constant), then
  // a CTA-local order: interior nodes first, boundary nodes last, each by descending degree
  // (small SELL padding). The partition is fixed before the reorder, which stays inside ranges.
  t.nslices = (n + 31) / 32;
  // one SM stays free for the v5 kernel's convergence-master CTA
  const int sms = sweep_grid_ctas(t.dev);
  const int target = t.partition_override > 0 ? t.partition_override
                     : g_sweep_partition > 0   ? g_sweep_partition
                                               : (sms > 1 ? sms - 1 : 1);
  t.sweep_ctas = (int)std::max<int64_t>(1, std::min<int64_t>(target, t.nslices));
  const int G = t.sweep_ctas;
  t.cta_lo.alloc(G + 1, s);
  t.cta_int_hi.alloc(G, s);
  if (n > 0) {
    DBuf<int64_t> w(t.nslices + 1, s), wp(t.nslices + 1, s);
    k_slice_weight<<<grid_for(t.nslices, 256), 256, 0, s>>>(n, t.nslices, t.deg.get(), w.get());
    launched("slice_weight");
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, w.get(), wp.get(), t.nslices + 1, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, w.get(), wp.get(), t.nslices + 1, s));
    launched("scan_weight");
    k_partition<<<grid_for(G + 1, 128), 128, 0, s>>>(G, t.nslices, wp.get(), t.cta_lo.get());
    launched("partition");
    DBuf<int32_t> cos(t.nslices, s);
    k_cta_of_slice<<<G, 128, 0, s>>>(G, t.cta_lo.get(), cos.get());
    launched("cta_of_slice");
    DBuf<uint8_t> bnd(n, s);
    F2M_CUDA(cudaMemsetAsync(bnd.get(), 0, n, s));
    if (m > 0) {
      k_boundary<<<grid_for(m, 256), 256, 0, s>>>(m, t.eu.get(), t.ev.get(), t.perm.get(), cos.get(), bnd.get());
      launched("boundary");
    }
    DBuf<uint64_t> k0(n, s), k1(n, s);
    DBuf<int32_t> v0(n, s), v1(n, s), deg2(n, s), ip2(n, s), p2(n, s), nint(G, s);
    F2M_CUDA(cudaMemsetAsync(nint.get(), 0, sizeof(int32_t) * G, s));
    constexpr int dbits = 7;  // degrees ordered exactly up to 127
    const int key_bits = bit_width(std::max(G - 1, 1)) + 1 + dbits;
    k_local_keys<<<grid_for(n, 256), 256, 0, s>>>(n, t.deg.get(), bnd.get(), cos.get(), dbits, (1 << dbits) - 1,
                                                 k0.get(), v0.get(), nint.get());
    launched("local_keys");
    tmp = 0;
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.get(), k1.get(), v0.get(), v1.get(), n, 0, key_bits, s));
    DBuf<char> tb2(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(tb2.get(), tmp, k0.get(), k1.get(), v0.get(), v1.get(), n, 0, key_bits,
                                             s));
    launched("sort_local");
    k_window_apply<<<grid_for(n, 256), 256, 0, s>>>(n, v1.get(), t.deg.get(), t.iperm.get(), deg2.get(), ip2.get(),
                                                   p2.get());
    launched("local_apply");
    t.deg = std::move(deg2);
    t.iperm = std::move(ip2);
    t.perm = std::move(p2);
    k_int_hi<<<grid_for(G, 128), 128, 0, s>>>(G, t.cta_lo.get(), nint.get(), t.cta_int_hi.get());
    launched("int_hi");
    t.cta_nint = std::move(nint);
  } else {
    int zero[2] = {0, 0};
    F2M_CUDA(cudaMemcpyAsync(t.cta_lo.get(), zero, sizeof(int32_t) * 2, cudaMemcpyHostToDevice, s));
    F2M_CUDA(cudaMemcpyAsync(t.cta_int_hi.get(), zero, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  }
  // min / max degree and the SELL-32 layout; their sizes come back with ONE synchronisation
  DBuf<int> mm(2, s);
  {
    int* init = reinterpret_cast<int*>(pinned_scratch());
    init[0] = n > 0 ? INT_MAX : 0;
    init[1] = 0;
    F2M_CUDA(cudaMemcpyAsync(mm.get(), init, 2 * sizeof(int), cudaMemcpyHostToDevice, s));
    if (n > 0) {
      k_minmax_deg<<<std::min<unsigned>(grid_for(n, 256), 1184), 256, 0, s>>>(n, t.deg.get(),
                                                                               mm.get(), mm.get() + 1);
      launched("minmax_deg");
    }
  }
  t.swidth.alloc(t.nslices, s);
  t.sptr.alloc(t.nslices + 1, s);
  DBuf<int64_t> ssize(t.nslices + 1, s);
  if (t.nslices > 0) {
    k_slice_width<<<grid_for(t.nslices, 256), 256, 0, s>>>(n, t.nslices, t.deg.get(), t.swidth.get(),
                                                          ssize.get());
    launched("slice_width");
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ssize.get(), t.sptr.get(), t.nslices + 1, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, ssize.get(), t.sptr.get(), t.nslices + 1, s));
    launched("scan_slices");
  } else {
    F2M_CUDA(cudaMemsetAsync(t.sptr.get(), 0, sizeof(int64_t), s));
  }
  // exclusive scan over nslices+1 entries: sptr[nslices] = total padded slots (the last
  // input entry never contributes to an exclusive sum)
  int64_t slots = 0;
  {
    int64_t* hs = pinned_scratch();
    F2M_CUDA(cudaMemcpyAsync(hs + 8, mm.get(), 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaMemcpyAsync(hs + 9, t.sptr.get() + t.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    const int* mmh = reinterpret_cast<const int*>(hs + 8);
    t.min_deg = mmh[0];
    t.max_deg = mmh[1];
    slots = hs[9];
  }
  t.sell_slots = slots;
  t.scol.alloc(slots, s);
  t.seid.alloc(slots, s);
  if (t.nslices > 0) {
    k_fill_pad<<<grid_for(t.nslices * 32, 256), 256, 0, s>>>(t.nslices, t.sptr.get(), t.scol.get(),
                                                            t.seid.get());
    launched("fill_pad");
  }
  if (m > 0) {
    DBuf<int32_t> fill(n, s);
    F2M_CUDA(cudaMemsetAsync(fill.get(), 0, sizeof(int32_t) * n, s));
    k_fill_sell<<<grid_for(m, 256), 256, 0, s>>>(m, t.eu.get(), t.ev.get(), t.perm.get(), t.sptr.get(),
                                                fill.get(), t.scol.get(), t.seid.get());
    launched("fill_sell");
  }
  build_local_index(t);
}

// Graph::from_edges mean (graph.cpp:47-49): a SEQUENTIAL fp64 sum in edge order divided by m. It
// sets the convergence threshold eps*mean_cost, so it must be bit-exact: seq_sums_device
// reproduces the left-to-right chain; the division is IEEE (correctly rounded) on the host.
double sequential_mean(const double* d_cost, int64_t m, cudaStream_t s) {
  if (m <= 0) return 0.0;
  DBuf<double> out(1, s);
  seq_sums_device(d_cost, m, m, out.get(), s);
  double h = 0.0;
  F2M_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  return h / (double)m;
}

void attach_costs(f2m_graph& g) {
  Topology& t = *g.topo;
  g.scost.alloc(t.sell_slots, t.stream);
  if (t.sell_slots > 0) {
    k_scost<<<grid_for(t.sell_slots, 256), 256, 0, t.stream>>>(t.sell_slots, t.seid.get(),
                                                               g.cost.get(), g.scost.get());
    launched("scost");
  }
  g.mean_known = false;
  g.approx_sum.alloc(1, t.stream);
  if (t.m > 0) {
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, g.cost.get(), g.approx_sum.get(), t.m, t.stream));
    DBuf<char> tb(tmp, t.stream);
    F2M_CUDA(cub::DeviceReduce::Sum(tb.get(), tmp, g.cost.get(), g.approx_sum.get(), t.m, t.stream));
    launched("approx_cost_sum");
  } else {
    F2M_CUDA(cudaMemsetAsync(g.approx_sum.get(), 0, sizeof(double), t.stream));
  }
}

double graph_mean(const f2m_graph& g) {
  if (!g.mean_known) {
    g.mean_cost = sequential_mean(g.cost.get(), g.topo->m, g.topo->stream);
    g.mean_known = true;
  }
  return g.mean_cost;
}

void upload_lambda(const f2m_graph& g, const double* h_lambda, double* d_lam_pos) {
  const Topology& t = *g.topo;
  if (t.n == 0) return;
  DBuf<double> tmp(t.n, t.stream);
  F2M_CUDA(cudaMemcpyAsync(tmp.get(), h_lambda, sizeof(double) * t.n, cudaMemcpyHostToDevice, t.stream));
  k_scatter_f64<<<grid_for(t.n, 256), 256, 0, t.stream>>>(t.n, tmp.get(), t.perm.get(), d_lam_pos);
  launched("scatter_lambda");
}

void download_lambda(const f2m_graph& g, const double* d_lam_pos, double* h_lambda) {
  const Topology& t = *g.topo;
  if (t.n == 0) return;
  DBuf<double> tmp(t.n, t.stream);
  k_gather_f64<<<grid_for(t.n, 256), 256, 0, t.stream>>>(t.n, d_lam_pos, t.perm.get(), tmp.get());
  launched("gather_lambda");
  F2M_CUDA(cudaMemcpyAsync(h_lambda, tmp.get(), sizeof(double) * t.n, cudaMemcpyDeviceToHost, t.stream));
  F2M_CUDA(cudaStreamSynchronize(t.stream));
}

}  // namespace f2mgpu

using namespace f2mgpu;

// ====================================================================== C ABI

extern "C" const char* f2m_last_error(void) { return t_last_error.c_str(); }

extern "C" int f2m_set_device(int device) {
  return guard([&] {
    int count = 0;
    F2M_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw Error(F2M_E_ARGUMENT, "f2m_set_device: no such device");
    F2M_CUDA(cudaSetDevice(device));
    t_device = device;
  });
}

extern "C" int f2m_get_device_info(f2m_device_info* out) {
  return guard([&] {
    const int dev = current_device();
    F2M_CUDA(cudaSetDevice(dev));
    const cudaDeviceProp& p = device_props(dev);
    out->device = dev;
    out->sm_count = p.multiProcessorCount;
    out->sweep_ctas = sweep_grid_ctas(dev);
    out->sweep_threads = sweep_block_threads();
    out->cc_major = p.major;
    out->cc_minor = p.minor;
    std::snprintf(out->name, sizeof(out->name), "%s", p.name);
  });
}

extern "C" uint64_t f2m_kernel_launch_count(void) { return g_launches.load(); }

extern "C" int f2m_graph_from_edges(int n, int64_t m, const int32_t* eu, const int32_t* ev,
                                    const double* cost, f2m_graph** out) {
  return guard([&] {
    *out = nullptr;
    if (n < 0) throw Error(F2M_E_ARGUMENT, "from_edges: negative node count");
    if (m < 0) throw Error(F2M_E_ARGUMENT, "from_edges: negative edge count");
    if (m >= (int64_t(1) << 30)) throw Error(F2M_E_ARGUMENT, "from_edges: too many edges");
    for (int64_t e = 0; e < m; ++e) {  // graph.cpp:16-19: IndexError before anything else
      if (eu[e] < 0 || eu[e] >= n || ev[e] < 0 || ev[e] >= n)
        throw Error(F2M_E_INDEX, "edge endpoint out of range");
    }
    const int dev = current_device();
    F2M_CUDA(cudaSetDevice(dev));
    auto g = std::make_unique<f2m_graph>();
    g->topo = make_topology(n, dev);
    Topology& t = *g->topo;
    t.m = m;
    cudaStream_t s = t.stream;
    DBuf<int32_t> du(m, s), dv(m, s);
    g->cost.alloc(m, s);
    if (m > 0) {
      F2M_CUDA(cudaMemcpyAsync(du.get(), eu, sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
      F2M_CUDA(cudaMemcpyAsync(dv.get(), ev, sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
      F2M_CUDA(cudaMemcpyAsync(g->cost.get(), cost, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    }
    sort_edges(t, du, dv, g->cost);
    identity_perm(t);
    finalize_topology(t);
    attach_costs(*g);
    F2M_CUDA(cudaStreamSynchronize(s));
    *out = g.release();
  });
}

extern "C" int f2m_graph_with_costs(const f2m_graph* g, const double* cost, f2m_graph** out) {
  return guard([&] {
    *out = nullptr;
    F2M_CUDA(cudaSetDevice(g->topo->dev));
    auto h = std::make_unique<f2m_graph>();
    h->topo = g->topo;
    const Topology& t = *h->topo;
    h->cost.alloc(t.m, t.stream);
    if (t.m > 0)
      F2M_CUDA(cudaMemcpyAsync(h->cost.get(), cost, sizeof(double) * t.m, cudaMemcpyHostToDevice, t.stream));
    attach_costs(*h);
    *out = h.release();
  });
}

extern "C" int f2m_graph_jittered(const f2m_graph* g, uint64_t seed, int restart,
                                  double perturb_scale, f2m_graph** out) {
  return guard([&] {
    *out = nullptr;
    F2M_CUDA(cudaSetDevice(g->topo->dev));
    auto h = std::make_unique<f2m_graph>();
    h->topo = g->topo;
    const Topology& t = *h->topo;
    // cost_scale (solve.cpp:33-35) and amplitude (:40) are host scalars, as in the reference
    const double scale = graph_mean(*g) > 0.0 ? g->mean_cost : 1.0;
    const double amplitude = perturb_scale * scale;
    const uint64_t state0 = seed * 0x9E3779B97F4A7C15ULL + static_cast<uint64_t>(restart);
    h->cost.alloc(t.m, t.stream);
    if (t.m > 0) {
      k_jitter<<<grid_for(t.m, 256), 256, 0, t.stream>>>(t.m, g->cost.get(), amplitude, state0,
                                                        h->cost.get());
      launched("jitter");
    }
    attach_costs(*h);
    *out = h.release();
  });
}

extern "C" void f2m_graph_destroy(f2m_graph* g) {
  if (!g) return;
  cudaSetDevice(g->topo->dev);
  delete g;
}

extern "C" int f2m_graph_get_info(const f2m_graph* g, f2m_graph_info* out) {
  return guard([&] {
    const Topology& t = *g->topo;
    out->n = t.n;
    out->m = t.m;
    out->mean_cost = graph_mean(*g);
    out->min_degree = t.min_deg;
    out->max_degree = t.max_deg;
    out->sell_slots = t.sell_slots;
    out->sweep_ctas = t.sweep_ctas;
    out->sweep_variant = !t.v2 ? 1 : (t.resident ? 3 : 2);
    out->max_local = t.max_local;
    out->max_cta_slots = t.max_cta_slots;
    out->smem_bytes = (int64_t)t.smem_bytes;
  });
}

extern "C" int f2m_graph_edges(const f2m_graph* g, int32_t* eu, int32_t* ev, double* cost) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.m > 0) {
      if (eu) F2M_CUDA(cudaMemcpyAsync(eu, t.eu.get(), sizeof(int32_t) * t.m, cudaMemcpyDeviceToHost, t.stream));
      if (ev) F2M_CUDA(cudaMemcpyAsync(ev, t.ev.get(), sizeof(int32_t) * t.m, cudaMemcpyDeviceToHost, t.stream));
      if (cost) F2M_CUDA(cudaMemcpyAsync(cost, g->cost.get(), sizeof(double) * t.m, cudaMemcpyDeviceToHost, t.stream));
    }
    F2M_CUDA(cudaStreamSynchronize(t.stream));
  });
}

extern "C" int f2m_graph_degrees(const f2m_graph* g, int32_t* degree) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.n == 0) return;
    DBuf<int32_t> tmp(t.n, t.stream);
    k_gather_i32<<<grid_for(t.n, 256), 256, 0, t.stream>>>(t.n, t.deg.get(), t.perm.get(), tmp.get());
    launched("gather_deg");
    F2M_CUDA(cudaMemcpyAsync(degree, tmp.get(), sizeof(int32_t) * t.n, cudaMemcpyDeviceToHost, t.stream));
    F2M_CUDA(cudaStreamSynchronize(t.stream));
  });
}

extern "C" int f2m_graph_incidence(const f2m_graph* g, int64_t* offsets, int32_t* ids) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    const int n = t.n;
    const int64_t m = t.m;
    DBuf<int32_t> deg(n, s);
    DBuf<int64_t> degl(n + 1, s), off(n + 1, s);
    if (n > 0) {
      k_gather_i32<<<grid_for(n, 256), 256, 0, s>>>(n, t.deg.get(), t.perm.get(), deg.get());
      launched("gather_deg");
    }
    std::vector<int32_t> hdeg(n);
    if (n > 0)
      F2M_CUDA(cudaMemcpyAsync(hdeg.data(), deg.get(), sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    offsets[0] = 0;
    for (int v = 0; v < n; ++v) offsets[v + 1] = offsets[v] + hdeg[v];
    const int64_t slots = offsets[n];
    DBuf<int32_t> d_ids(slots, s), cur(n, s);
    if (n > 0) {
      F2M_CUDA(cudaMemcpyAsync(off.get(), offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
      F2M_CUDA(cudaMemsetAsync(cur.get(), 0, sizeof(int32_t) * n, s));
    }
    if (m > 0) {
      k_incidence_keys<<<grid_for(m, 256), 256, 0, s>>>(m, t.eu.get(), t.ev.get(), off.get(), cur.get(),
                                                       d_ids.get());
      launched("incidence");
    }
    if (slots > 0)
      F2M_CUDA(cudaMemcpyAsync(ids, d_ids.get(), sizeof(int32_t) * slots, cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    // rows hold ascending edge ids in the reference (graph.cpp:38-44)
    for (int v = 0; v < n; ++v) std::sort(ids + offsets[v], ids + offsets[v + 1]);
  });
}

namespace f2mgpu {
// validate_graph (graph.cpp:242-277) on the device: the first defect's {edge << 2 | kind} goes to
// the page-locked *h_first (all ones: none) without a synchronisation
void validate_graph_async(const f2m_graph& g, unsigned long long* h_first) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  *h_first = ~0ULL;
  if (t.m <= 0) return;
  DBuf<unsigned long long> first(1, s);
  F2M_CUDA(cudaMemsetAsync(first.get(), 0xff, sizeof(unsigned long long), s));
  k_validate<<<grid_for(t.m, 256), 256, 0, s>>>(t.m, t.eu.get(), t.ev.get(), g.cost.get(), first.get());
  launched("validate");
  F2M_CUDA(cudaMemcpyAsync(h_first, first.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
}
// after a synchronisation of the graph's stream: throw the defect validate_graph_async found
void validate_graph_check(const f2m_graph& g, unsigned long long h) {
  if (h == ~0ULL) return;
  const Topology& t = *g.topo;
  const int64_t e = (int64_t)(h >> 2);
  const int kind = (int)(h & 3);
  int32_t u = 0, v = 0;
  F2M_CUDA(cudaMemcpy(&u, t.eu.get() + e, sizeof(int32_t), cudaMemcpyDeviceToHost));
  F2M_CUDA(cudaMemcpy(&v, t.ev.get() + e, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (kind == 1) throw Error(F2M_E_STRUCTURE, "self-loop at node " + std::to_string(u));
  if (kind == 2) throw Error(F2M_E_STRUCTURE, "duplicate edge (" + std::to_string(u) + ", " + std::to_string(v) + ")");
  throw Error(F2M_E_STRUCTURE, "negative cost on edge (" + std::to_string(u) + ", " + std::to_string(v) + ")");
}
}  // namespace f2mgpu

extern "C" int f2m_graph_validate(const f2m_graph* g, int* min_degree, int* max_degree,
                                  int64_t* edges) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    unsigned long long* hf = reinterpret_cast<unsigned long long*>(pinned_scratch() + 15);
    validate_graph_async(*g, hf);
    F2M_CUDA(cudaStreamSynchronize(t.stream));
    validate_graph_check(*g, *hf);
    const int mn = t.n > 0 ? t.min_deg : 0;
    if (min_degree) *min_degree = mn;
    if (max_degree) *max_degree = t.max_deg;
    if (edges) *edges = t.m;
    if (mn < 3)
      throw Error(F2M_E_MIN_DEGREE, "node degree " + std::to_string(mn) +
                                        " below 3; the node update needs a third-shortest edge");
  });
}

extern "C" double f2m_sweep_algorithmic_bytes(const f2m_graph* g) {
  const Topology& t = *g->topo;
  return 4.0 * (t.n + 1) + 2.0 * t.m * 12.0 + 16.0 * t.n;
}


extern "C" void f2m_set_sweep_partition(int ctas) { f2mgpu::g_sweep_partition = ctas > 0 ? ctas : 0; }

// knn.cu — grid-bucketed k-nearest-neighbour candidate graph (build_knn_graph,
// graph.cpp:169-240) on sm_100a.
//
// One thread per query replays the reference's ring expansion over the SAME PointGrid
// (graph.cpp:79-116: bbox, cell = sqrt(area/n) doubled until gx*gy <= 64+8n) with the SAME
// exact stop bound (graph.cpp:203-211). The kept set — the per_node smallest (d, idx) pairs
// among the candidates offered — does not depend on the order candidates are offered, so the
// within-cell order of the bucketing (atomics here) is free and the candidate lists are
// bit-identical to the reference's. Symmetrization is a 64-bit radix sort + unique over
// (min, max) keys (graph.cpp:223-232); costs are distance(u, v) with no FMA
// (instance.cpp:134-136). The device node order is the Morton (Z) order of grid cells, which
// makes a CTA's slice range a compact spatial patch for the sweep's lambda gathers.
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "internal.cuh"

namespace f2mgpu {

struct GridParams {
  double min_x, max_x, min_y, max_y;
  double cell;
  int gx, gy;
  int max_ring;
};

__device__ __forceinline__ unsigned long long dkey(double v) {
  // monotone map double -> u64 (finite values)
  unsigned long long b = __double_as_longlong(v);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double(b);
}

__global__ void k_bbox(int n, const double* __restrict__ xy, unsigned long long* __restrict__ acc) {
  // acc[0] = min x key, acc[1] = max x key, acc[2] = min y, acc[3] = max y
  unsigned long long mnx = ~0ULL, mxx = 0, mny = ~0ULL, mxy = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long kx = dkey(xy[2 * i]), ky = dkey(xy[2 * i + 1]);
    mnx = min(mnx, kx); mxx = max(mxx, kx);
    mny = min(mny, ky); mxy = max(mxy, ky);
  }
  for (int o = 16; o; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&acc[0], mnx); atomicMax(&acc[1], mxx);
    atomicMin(&acc[2], mny); atomicMax(&acc[3], mxy);
  }
}

// PointGrid constructor arithmetic (graph.cpp:79-101), one thread.
__global__ void k_grid_params(int n, const unsigned long long* __restrict__ acc, GridParams* gp) {
  GridParams p;
  p.min_x = dkey_inv(acc[0]); p.max_x = dkey_inv(acc[1]);
  p.min_y = dkey_inv(acc[2]); p.max_y = dkey_inv(acc[3]);
  const double width = dsub(p.max_x, p.min_x);
  const double height = dsub(p.max_y, p.min_y);
  const double area = dmul(width, height);
  double cell = area > 0.0 ? __dsqrt_rn(__ddiv_rn(area, (double)n)) : (width < height ? height : width);
  if (!(cell > 0.0)) cell = 1.0;
  int gx, gy;
  for (;;) {
    gx = max(1, __double2int_rz(__ddiv_rn(width, cell)) + 1);
    gy = max(1, __double2int_rz(__ddiv_rn(height, cell)) + 1);
    if ((long long)gx * gy <= 64 + 8 * (long long)n) break;
    cell = dmul(cell, 2.0);
  }
  p.cell = cell;
  p.gx = gx;
  p.gy = gy;
  p.max_ring = max(gx, gy);
  *gp = p;
}

__device__ __forceinline__ int clamp_c(double v, double lo, double cell, int g) {
  // static_cast<int>((x - min_x) / cell) clamped to [0, g-1] (graph.cpp:118-125)
  const int c = __double2int_rz(__ddiv_rn(dsub(v, lo), cell));
  return min(max(c, 0), g - 1);
}

__global__ void k_cell_hist(int n, const double* __restrict__ xy, const GridParams* __restrict__ gp,
                            int32_t* __restrict__ cell_of, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const GridParams p = *gp;
  const int cx = clamp_c(xy[2 * i], p.min_x, p.cell, p.gx);
  const int cy = clamp_c(xy[2 * i + 1], p.min_y, p.cell, p.gy);
  const int c = cy * p.gx + cx;
  cell_of[i] = c;
  atomicAdd(&cnt[c], 1);
}

__global__ void k_cell_scatter(int n, const double* __restrict__ xy, const int32_t* __restrict__ cell_of,
                               const int32_t* __restrict__ off, int32_t* __restrict__ cur,
                               int32_t* __restrict__ ids, double2* __restrict__ pts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_of[i];
  const int t = off[c] + atomicAdd(&cur[c], 1);
  ids[t] = i;
  pts[t] = make_double2(xy[2 * i], xy[2 * i + 1]);
}

__device__ __forceinline__ double point_distance(double ax, double ay, double bx, double by,
                                                 int rounded) {
  // distance(): sqrt(dx*dx + dy*dy), rounded -> floor(d + 0.5)  (instance.cpp:134-139)
  const double dx = dsub(ax, bx);
  const double dy = dsub(ay, by);
  const double d = __dsqrt_rn(dadd(dmul(dx, dx), dmul(dy, dy)));
  return rounded ? floor(dadd(d, 0.5)) : d;
}

// Bounded sorted list of the best (d, idx) pairs — NeighborHeap (graph.cpp:135-165) semantics.
template <int KMAX>
struct Best {
  double d[KMAX > 0 ? KMAX : 1];
  int id[KMAX > 0 ? KMAX : 1];
};

template <int KMAX>
__global__ void __launch_bounds__(128) k_knn_query(int n, int per_node, int rounded,
                                                   const double* __restrict__ xy,
                                                   const GridParams* __restrict__ gpp,
                                                   const int32_t* __restrict__ off,
                                                   const int32_t* __restrict__ ids,
                                                   const double2* __restrict__ pts,
                                                   double* __restrict__ scratch_d,
                                                   int* __restrict__ scratch_i,
                                                   int32_t* __restrict__ nbr) {
  // queries run in cell order (ids / pts are the points sorted by grid cell): the lanes of a warp
  // scan overlapping neighbourhoods (L1 reuse, similar trip counts); results go to the node's row
  const int tq = blockIdx.x * blockDim.x + threadIdx.x;
  if (tq >= n) return;
  const int node = ids[tq];
  const GridParams p = *gpp;
  Best<KMAX> local;
  double* hd = KMAX > 0 ? local.d : scratch_d + (int64_t)node * per_node;
  int* hi = KMAX > 0 ? local.id : scratch_i + (int64_t)node * per_node;
  int cnt = 0;
  const double2 self = pts[tq];
  const double ax = self.x, ay = self.y;
  const int ccx = clamp_c(ax, p.min_x, p.cell, p.gx);
  const int ccy = clamp_c(ay, p.min_y, p.cell, p.gy);
  for (int r = 0; r <= p.max_ring; ++r) {
    const int x0 = ccx - r, x1 = ccx + r, y0 = ccy - r, y1 = ccy + r;
    const int ylo = max(0, y0), yhi = min(p.gy - 1, y1);
    const int xlo = max(0, x0), xhi = min(p.gx - 1, x1);
    auto visit = [&](int cx, int cy) {
      const int c = cy * p.gx + cx;
      for (int t = off[c]; t < off[c + 1]; ++t) {
        const int q = ids[t];
        if (q == node) continue;
        const double2 b = pts[t];
        const double dd = point_distance(ax, ay, b.x, b.y, rounded);
        if (cnt == per_node) {
          if (!(dd < hd[per_node - 1] || (dd == hd[per_node - 1] && q < hi[per_node - 1]))) continue;
          --cnt;
        }
        int i = cnt++;
        while (i > 0 && (hd[i - 1] > dd || (hd[i - 1] == dd && hi[i - 1] > q))) {
          hd[i] = hd[i - 1];
          hi[i] = hi[i - 1];
          --i;
        }
        hd[i] = dd;
        hi[i] = q;
      }
    };
    for (int cy = ylo; cy <= yhi; ++cy) {
      if (cy == y0 || cy == y1) {  // ring cells only (graph.cpp:212-214)
        for (int cx = xlo; cx <= xhi; ++cx) visit(cx, cy);
      } else {
        if (x0 >= 0) visit(x0, cy);
        if (x1 <= p.gx - 1) visit(x1, cy);
      }
    }
    if (cnt == per_node) {
      // unseen points are at distance >= r*cell; exact bound of graph.cpp:203-211
      double bound = dmul(dmul((double)r, p.cell), 1.0 - 1e-12);
      if (rounded) bound = dsub(bound, 0.5);
      if (bound > hd[per_node - 1]) break;
    }
  }
  for (int j = 0; j < per_node; ++j) nbr[(int64_t)node * per_node + j] = hi[j];
}

// Fixed-K variant (K = per_node known at compile time): the sorted top-K list lives in
// registers (fully unrolled insertion, no local memory). Same candidates, same (distance, id)
// total order and the same ring-termination bound as k_knn_query -> identical lists.
template <int K>
__global__ void __launch_bounds__(128, 4) k_knn_query_reg(int n, int rounded, const GridParams* __restrict__ gpp,
                                                       const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ ids,
                                                       const double2* __restrict__ pts,
                                                       int32_t* __restrict__ nbr) {
  const int tq = blockIdx.x * blockDim.x + threadIdx.x;  // cell order (see k_knn_query)
  if (tq >= n) return;
  const int node = ids[tq];
  const GridParams p = *gpp;
  double hd[K];
  int hi[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    hd[j] = CUDART_INF;
    hi[j] = INT_MAX;
  }
  const double2 self = pts[tq];
  const double ax = self.x, ay = self.y;
  const int ccx = clamp_c(ax, p.min_x, p.cell, p.gx);
  const int ccy = clamp_c(ay, p.min_y, p.cell, p.gy);
  auto visit = [&](int cx, int cy) {
    const int c = cy * p.gx + cx;
    const int t1 = off[c + 1];
    for (int t = off[c]; t < t1; ++t) {
      const int q = ids[t];
      if (q == node) continue;
      const double2 b = pts[t];
      const double dd = point_distance(ax, ay, b.x, b.y, rounded);
      if (!(dd < hd[K - 1] || (dd == hd[K - 1] && q < hi[K - 1]))) continue;
      bool placed = false;
#pragma unroll
      for (int j = K - 1; j > 0; --j) {
        const bool lt = dd < hd[j - 1] || (dd == hd[j - 1] && q < hi[j - 1]);
        const double nd = lt ? hd[j - 1] : (placed ? hd[j] : dd);
        const int ni = lt ? hi[j - 1] : (placed ? hi[j] : q);
        hd[j] = nd;
        hi[j] = ni;
        placed = placed || !lt;
      }
      if (!placed) {
        hd[0] = dd;
        hi[0] = q;
      }
    }
  };
  for (int r = 0; r <= p.max_ring; ++r) {
    const int x0 = ccx - r, x1 = ccx + r, y0 = ccy - r, y1 = ccy + r;
    const int ylo = max(0, y0), yhi = min(p.gy - 1, y1);
    const int xlo = max(0, x0), xhi = min(p.gx - 1, x1);
    for (int cy = ylo; cy <= yhi; ++cy) {
      if (cy == y0 || cy == y1) {  // ring cells only (graph.cpp:212-214)
        for (int cx = xlo; cx <= xhi; ++cx) visit(cx, cy);
      } else {
        if (x0 >= 0) visit(x0, cy);
        if (x1 <= p.gx - 1) visit(x1, cy);
      }
    }
    if (hi[K - 1] != INT_MAX) {  // K found; unseen points are at distance >= r*cell (graph.cpp:203-211)
      double bound = dmul(dmul((double)r, p.cell), 1.0 - 1e-12);
      if (rounded) bound = dsub(bound, 0.5);
      if (bound > hd[K - 1]) break;
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) nbr[(int64_t)node * K + j] = hi[j];
}

__global__ void k_pair_keys(int n, int per_node, int bits, const int32_t* __restrict__ nbr,
                            uint64_t* __restrict__ keys) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * per_node) return;
  const int i = (int)(t / per_node);
  const int q = nbr[t];
  const uint32_t a = (uint32_t)min(i, q), b = (uint32_t)max(i, q);
  keys[t] = ((uint64_t)a << bits) | b;  // (min, max) packed into 2*bits bits: short radix sort
}

__global__ void k_edges_from_keys(int64_t m, const uint64_t* __restrict__ keys, int bits,
                                  const double* __restrict__ xy, int rounded,
                                  int32_t* __restrict__ eu, int32_t* __restrict__ ev,
                                  double* __restrict__ cost) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int u = (int)(keys[e] >> bits), v = (int)(keys[e] & ((1ull << bits) - 1));
  eu[e] = u;
  ev[e] = v;
  cost[e] = point_distance(xy[2 * u], xy[2 * u + 1], xy[2 * v], xy[2 * v + 1], rounded);
}

__device__ __forceinline__ uint64_t spread32(uint32_t v) {
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFULL;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFULL;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0FULL;
  x = (x | (x << 2)) & 0x3333333333333333ULL;
  x = (x | (x << 1)) & 0x5555555555555555ULL;
  return x;
}

// Hilbert index of cell (x, y) on a 2^order x 2^order grid (the classic rotate-and-flip walk):
// consecutive Hilbert ranges are compact patches without Morton's long jumps, so the sweep
// kernel's CTA partitions have fewer boundary rows and neighbour CTAs.
__device__ __forceinline__ uint64_t hilbert_d(int order, uint32_t x, uint32_t y) {
  uint64_t d = 0;
  for (uint32_t sside = 1u << (order - 1); sside > 0; sside >>= 1) {
    const uint32_t rx = (x & sside) ? 1u : 0u, ry = (y & sside) ? 1u : 0u;
    d += (uint64_t)sside * sside * ((3u * rx) ^ ry);
    if (ry == 0) {  // rotate the quadrant
      if (rx == 1) {
        x = sside - 1 - (x & (sside - 1)) + (x & ~(sside - 1));
        y = sside - 1 - (y & (sside - 1)) + (y & ~(sside - 1));
      }
      const uint32_t t = x;
      x = y;
      y = t;
    }
  }
  return d;
}

__global__ void k_morton(int n, const int32_t* __restrict__ cell_of, const GridParams* __restrict__ gp, int order,
                         int hilbert, uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_of[i];
  const int gx = gp->gx;
  const uint32_t cx = (uint32_t)(c % gx), cy = (uint32_t)(c / gx);
  key[i] = hilbert ? hilbert_d(order, cx, cy) : (spread32(cx) | (spread32(cy) << 1));
  idx[i] = i;
}

__global__ void k_points_by_position(int n, const double* __restrict__ xy, const int32_t* __restrict__ iperm,
                                     double2* __restrict__ pts) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const int v = iperm[p];
    pts[p] = make_double2(xy[2 * v], xy[2 * v + 1]);
  }
}

__global__ void k_invert(int n, const int32_t* __restrict__ iperm, int32_t* __restrict__ perm) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) perm[iperm[p]] = p;
}

f2m_graph* knn_build_device(int n, const double* xy, bool xy_on_host, int rounded, int k, int dev,
                            cudaEvent_t start) {
  if (k < 3) throw Error(F2M_E_ARGUMENT, "build_knn_graph: k must be >= 3");
  if (n < 4) throw Error(F2M_E_ARGUMENT, "build_knn_graph: need at least 4 nodes");
  const int per_node = std::min(k, n - 1);
  if ((int64_t)n * per_node >= (int64_t(1) << 31)) throw Error(F2M_E_ARGUMENT, "build_knn_graph: n*k too large");
  auto g = std::make_unique<f2m_graph>();
  g->topo = make_topology(n, dev);
  Topology& t = *g->topo;
  cudaStream_t s = t.stream;
  if (start) F2M_CUDA(cudaEventRecord(start, s));
  DBuf<double> staged;
  const double* d_xy = xy;
  if (xy_on_host) {
    staged.alloc(2 * (int64_t)n, s);
    F2M_CUDA(cudaMemcpyAsync(staged.get(), xy, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s));
    d_xy = staged.get();
  }

  // ---- PointGrid (graph.cpp:79-116)
  DBuf<unsigned long long> acc(4, s);
  unsigned long long init[4] = {~0ULL, 0ULL, ~0ULL, 0ULL};
  F2M_CUDA(cudaMemcpyAsync(acc.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_bbox<<<std::min<unsigned>(grid_for(n, 256), 2 * 148), 256, 0, s>>>(n, d_xy, acc.get());
  launched("bbox");
  DBuf<GridParams> gp(1, s);
  k_grid_params<<<1, 1, 0, s>>>(n, acc.get(), gp.get());
  launched("grid_params");
  GridParams hp;
  static_assert(sizeof(GridParams) <= 8 * sizeof(int64_t), "pinned scratch slots 50-57");
  // the grid's dimensions come back with the edge count's synchronisation below; until then the
  // cell arrays are sized by k_grid_params' bound gx * gy <= 64 + 8n (the unused cells stay empty)
  F2M_CUDA(cudaMemcpyAsync(pinned_scratch() + 50, gp.get(), sizeof(hp), cudaMemcpyDeviceToHost, s));
  const int64_t cells = 64 + 8 * (int64_t)n;
  DBuf<int32_t> cell_of(n, s), cnt(cells + 1, s), off(cells + 1, s), cur(cells, s), ids(n, s);
  DBuf<double2> pts(n, s);
  F2M_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (cells + 1), s));
  F2M_CUDA(cudaMemsetAsync(cur.get(), 0, sizeof(int32_t) * cells, s));
  k_cell_hist<<<grid_for(n, 256), 256, 0, s>>>(n, d_xy, gp.get(), cell_of.get(), cnt.get());
  launched("cell_hist");
  {
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), off.get(), cells + 1, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, cnt.get(), off.get(), cells + 1, s));
    launched("cell_scan");
  }
  k_cell_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, d_xy, cell_of.get(), off.get(), cur.get(), ids.get(),
                                                  pts.get());
  launched("cell_scatter");

  // ---- per-query ring search (graph.cpp:183-221)
  DBuf<int32_t> nbr((int64_t)n * per_node, s);
  DBuf<double> sd;
  DBuf<int> si;
  const unsigned qg = grid_for(n, 128);
  if (per_node >= 3 && per_node <= 12) {
    switch (per_node) {
#define F2M_KQ(K) \
  case K: k_knn_query_reg<K><<<qg, 128, 0, s>>>(n, rounded, gp.get(), off.get(), ids.get(), pts.get(), nbr.get()); break;
      F2M_KQ(3) F2M_KQ(4) F2M_KQ(5) F2M_KQ(6) F2M_KQ(7) F2M_KQ(8) F2M_KQ(9) F2M_KQ(10) F2M_KQ(11) F2M_KQ(12)
#undef F2M_KQ
    }
  } else if (per_node <= 16) {
    k_knn_query<16><<<qg, 128, 0, s>>>(n, per_node, rounded, d_xy, gp.get(), off.get(), ids.get(), pts.get(),
                                       nullptr, nullptr, nbr.get());
  } else if (per_node <= 32) {
    k_knn_query<32><<<qg, 128, 0, s>>>(n, per_node, rounded, d_xy, gp.get(), off.get(), ids.get(), pts.get(),
                                       nullptr, nullptr, nbr.get());
  } else {
    sd.alloc((int64_t)n * per_node, s);
    si.alloc((int64_t)n * per_node, s);
    k_knn_query<0><<<qg, 128, 0, s>>>(n, per_node, rounded, d_xy, gp.get(), off.get(), ids.get(), pts.get(),
                                      sd.get(), si.get(), nbr.get());
  }
  launched("knn_query");

  // ---- symmetrize: sort + unique (graph.cpp:223-232)
  const int64_t np = (int64_t)n * per_node;
  DBuf<uint64_t> k0(np, s), k1(np, s);
  int bits = 1;  // ids < 2^bits
  while ((1LL << bits) < n) ++bits;
  k_pair_keys<<<grid_for(np, 256), 256, 0, s>>>(n, per_node, bits, nbr.get(), k0.get());
  launched("pair_keys");
  {
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0.get(), k1.get(), np, 0, 2 * bits, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k0.get(), k1.get(), np, 0, 2 * bits, s));
    launched("sort_pairs");
  }
  DBuf<int64_t> nsel(1, s);
  {
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, k1.get(), k0.get(), nsel.get(), np, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceSelect::Unique(tb.get(), tmp, k1.get(), k0.get(), nsel.get(), np, s));
    launched("unique_pairs");
  }
  int64_t m = 0;
  F2M_CUDA(cudaMemcpyAsync(pinned_scratch() + 58, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  m = pinned_scratch()[58];
  std::memcpy(&hp, pinned_scratch() + 50, sizeof(hp));  // copied before the synchronisation above
  t.m = m;
  t.eu.alloc(m, s);
  t.ev.alloc(m, s);
  g->cost.alloc(m, s);
  k_edges_from_keys<<<grid_for(m, 256), 256, 0, s>>>(m, k0.get(), bits, d_xy, rounded, t.eu.get(), t.ev.get(),
                                                    g->cost.get());
  launched("edges_from_keys");

  // ---- spatial device order: Morton order of grid cells, ids ascending within a cell
  {
    DBuf<uint64_t> mk0(n, s), mk1(n, s);
    DBuf<int32_t> i0(n, s);
    t.iperm.alloc(n, s);
    t.perm.alloc(n, s);
    const int order = std::max(bit_width(std::max(hp.gx, hp.gy) - 1), 1);
    static const int hilbert = [] {
      const char* e = std::getenv("F2M_ORDER");
      return (e && e[0] == 'm') ? 0 : 1;  // F2M_ORDER=morton for A/B
    }();
    k_morton<<<grid_for(n, 256), 256, 0, s>>>(n, cell_of.get(), gp.get(), order, hilbert, mk0.get(), i0.get());
    launched("spatial_order");
    size_t tmp = 0;
    const int mbits = 2 * order;  // both curves index a 2^order x 2^order grid
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, mk0.get(), mk1.get(), i0.get(), t.iperm.get(), n,
                                             0, mbits, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, mk0.get(), mk1.get(), i0.get(), t.iperm.get(), n,
                                             0, mbits, s));
    launched("sort_morton");
    k_invert<<<grid_for(n, 256), 256, 0, s>>>(n, t.iperm.get(), t.perm.get());
    launched("invert_perm");
  }
  finalize_topology(t);
  attach_costs(*g);
  if (per_node == n - 1) {  // complete graph: keep the points for the all-pairs sweep
    g->pts_pos.alloc(n, s);
    k_points_by_position<<<grid_for(n, 256), 256, 0, s>>>(n, d_xy, t.iperm.get(), g->pts_pos.get());
    launched("points_by_position");
    g->rounded = rounded;
    g->allpairs = true;
  }
  return g.release();
}

}  // namespace f2mgpu

using namespace f2mgpu;

namespace f2mgpu {
// generate_instance (instance.cpp:143-157): point i takes draws 2i (x) and 2i+1 (y) of the
// SplitMix64 stream seeded `seed`, each next_double() * box (one rounded product: bit-exact).
__global__ void k_generate_uniform(int n, uint64_t seed, double box, double* __restrict__ xy) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= 2 * (int64_t)n) return;
  xy[j] = dmul(splitmix64_double_at(seed, (uint64_t)j), box);
}
}  // namespace f2mgpu

extern "C" int f2m_generate_instance_device(int n, uint64_t seed, double box, double* d_xy, void* stream) {
  return guard([&] {
    if (n < 1) throw Error(F2M_E_ARGUMENT, "generate_instance: n must be >= 1");
    if (!(box > 0.0)) throw Error(F2M_E_ARGUMENT, "generate_instance: box must be > 0");
    F2M_CUDA(cudaSetDevice(current_device()));
    k_generate_uniform<<<grid_for(2 * (int64_t)n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, seed, box,
                                                                                                     d_xy);
    launched("generate_uniform");
  });
}

extern "C" int f2m_knn_build_device(int n, const double* d_xy, int rounded, int k, f2m_graph** out) {
  return guard([&] {
    *out = nullptr;
    *out = knn_build_device(n, d_xy, false, rounded, k, current_device(), nullptr);
  });
}

extern "C" int f2m_knn_build(int n, const double* xy, int rounded, int k, f2m_graph** out) {
  return guard([&] {
    *out = nullptr;
    *out = knn_build_device(n, xy, true, rounded, k, current_device(), nullptr);
  });
}

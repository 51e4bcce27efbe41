// primal.cu — sign-pattern extraction and duality certificate on sm_100a (primal.cpp).
//
//  classify      k_classify: v_e = (c - l_u) - l_v (u < v) against [-tol, tol] (primal.cpp:43-63)
//                fused with the NEG / ZERO degree counts (primal.cpp:147-157).
//  degeneracy    first failing node in id order, same messages (primal.cpp:159-174).
//  components    lock-free union-find over the ZERO band that links the larger root under
//                the smaller (root = min node id, exactly the reference's DisjointSets result,
//                primal.cpp:20-39); zero edges sorted by (root, edge id) give every component
//                its edges in ascending id order (primal.cpp:179-194).
//  completion    one thread per component runs the reference's exhaustive DFS
//                (solve_zero_component, primal.cpp:65-140) iteratively, same visiting order,
//                same "first minimum wins" pruning -> identical x.
//  objective     sequential fp64 sum in edge order (primal.cpp:226-230), reproduced bit-exactly
//                by the parallel exact-sequential-sum primitive (seqsum.cu).
//  verify        per-node sums over the SELL rows (all partial sums are exact multiples of
//                1/2), value-set check, gap = objective - g(lambda) (primal.cpp:235-276).
#include <cstring>

#include <cub/cub.cuh>

#include "internal.cuh"

namespace f2mgpu {

__global__ void k_classify(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                           const double* __restrict__ cost, const int32_t* __restrict__ perm,
                           const double* __restrict__ lam, double tol, uint8_t* __restrict__ label,
                           int32_t* __restrict__ negd, int32_t* __restrict__ zerod,
                           double* __restrict__ x, uint8_t* __restrict__ zflag) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int u = eu[e], v = ev[e];
  const double val = dsub(dsub(cost[e], lam[perm[u]]), lam[perm[v]]);
  const uint8_t lab = val < -tol ? 0 : (val > tol ? 2 : 1);
  label[e] = lab;
  if (negd) {
    if (lab == 0) {
      atomicAdd(&negd[u], 1);
      atomicAdd(&negd[v], 1);
    } else if (lab == 1) {
      atomicAdd(&zerod[u], 1);
      atomicAdd(&zerod[v], 1);
    }
  }
  if (x) x[e] = lab == 0 ? 1.0 : 0.0;
  if (zflag) zflag[e] = lab == 1;
}

__global__ void k_check_nodes(int n, const int32_t* __restrict__ negd, const int32_t* __restrict__ zerod,
                              int32_t* __restrict__ residual, unsigned long long* __restrict__ first_bad) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int r = 2 - negd[v];
  residual[v] = r;
  if (negd[v] > 2) atomicMin(first_bad, (unsigned long long)v * 2);
  else if (r > 0 && zerod[v] == 0) atomicMin(first_bad, (unsigned long long)v * 2 + 1);
}

__global__ void k_iota_n(int n, int32_t* __restrict__ a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__device__ __forceinline__ int uf_find(int* parent, int x) {
  for (;;) {
    const int p = __ldcg(parent + x);
    if (p == x) return x;
    const int gp = __ldcg(parent + p);
    if (gp != p) atomicCAS(parent + x, p, gp);  // path halving, never changes the root set
    x = p;
  }
}

__global__ void k_union(int64_t z, const int32_t* __restrict__ zedges, const int32_t* __restrict__ eu,
                        const int32_t* __restrict__ ev, int* parent) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= z) return;
  const int e = zedges[i];
  int a = eu[e], b = ev[e];
  for (;;) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }
    // link the larger root under the smaller one (primal.cpp:31-34)
    if (atomicCAS(parent + b, b, a) == b) return;
  }
}

__global__ void k_comp_keys(int64_t z, const int32_t* __restrict__ zedges, const int32_t* __restrict__ eu,
                            int* parent, int ebits, uint64_t* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= z) return;
  const int e = zedges[i];
  // (component root, edge id) packed into bits(n) + ebits bits: short radix sort
  keys[i] = ((uint64_t)(uint32_t)uf_find(parent, eu[e]) << ebits) | (uint32_t)e;
}

__global__ void k_heads(int64_t z, const uint64_t* __restrict__ keys, int ebits, uint8_t* __restrict__ head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= z) return;
  head[i] = (i == 0) || ((keys[i] >> ebits) != (keys[i - 1] >> ebits));
}

// solve_zero_component (primal.cpp:65-140) as an iterative DFS with the recursion's exact
// visiting order and pruning. The search can be split: `depth` leading edges are forced to the
// base-3 digits of `prefix` (edge 0 most significant) and only that subtree is searched, with its
// own incumbent. The DFS keeps the FIRST leaf (in DFS = lexicographic order of the halves) that
// reaches the subtree's minimum — a later leaf of equal cost is pruned by `cost >= best` — so the
// whole search's answer is the minimum over subtrees of (cost, prefix): what k_components' warp
// reduction takes. Returns the subtree's best cost (+inf: none) and its halves in best[].
struct ZeroComponent {
  int mc, nn;
  int ce[kMaxComponentEdges];
  int ea[kMaxComponentEdges], eb[kMaxComponentEdges];
  double c[kMaxComponentEdges];
  int target[2 * kMaxComponentEdges];  // 2 x residual per local node
};

__device__ void component_setup(ZeroComponent& z, const int32_t* comp, int mc, const int32_t* __restrict__ eu,
                                const int32_t* __restrict__ ev, const double* __restrict__ cost,
                                const int32_t* __restrict__ residual, bool comp_is_sorted_keys,
                                const uint64_t* keys, int ebits) {
  int nodes[2 * kMaxComponentEdges];
  int nn = 0;
  z.mc = mc;
  for (int i = 0; i < mc; ++i) {
    z.ce[i] = comp_is_sorted_keys ? (int)(keys[i] & ((1ull << ebits) - 1)) : comp[i];
    nodes[nn++] = eu[z.ce[i]];
    nodes[nn++] = ev[z.ce[i]];
  }
  for (int i = 1; i < nn; ++i) {  // sort + unique (primal.cpp:73-75)
    const int v = nodes[i];
    int j = i;
    while (j > 0 && nodes[j - 1] > v) { nodes[j] = nodes[j - 1]; --j; }
    nodes[j] = v;
  }
  int u = 0;
  for (int i = 0; i < nn; ++i)
    if (i == 0 || nodes[i] != nodes[i - 1]) nodes[u++] = nodes[i];
  nn = u;
  z.nn = nn;
  auto local = [&](int v) {
    int lo = 0, hi = nn;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (nodes[mid] < v) lo = mid + 1; else hi = mid; }
    return lo;
  };
  for (int i = 0; i < nn; ++i) z.target[i] = 2 * residual[nodes[i]];
  for (int i = 0; i < mc; ++i) {
    z.ea[i] = local(eu[z.ce[i]]);
    z.eb[i] = local(ev[z.ce[i]]);
    z.c[i] = cost[z.ce[i]];
  }
}

__device__ double component_search(const ZeroComponent& z, int depth, int prefix, int* best) {
  const int mc = z.mc;
  int target[2 * kMaxComponentEdges], rem[2 * kMaxComponentEdges];
  int halves[kMaxComponentEdges];
  double cst[kMaxComponentEdges + 1];
  int hh[kMaxComponentEdges + 1];
  for (int i = 0; i < z.nn; ++i) { target[i] = z.target[i]; rem[i] = 0; }
  for (int i = 0; i < mc; ++i) {
    ++rem[z.ea[i]];
    ++rem[z.eb[i]];
    halves[i] = 0;
  }
  // the forced prefix: the same checks the DFS applies on its way down (LOOP below)
  cst[0] = 0.0;
  int pw = 1;
  for (int i = 1; i < depth; ++i) pw *= 3;
  for (int i = 0; i < depth; ++i, pw /= 3) {
    const int h = (prefix / pw) % 3, a = z.ea[i], b = z.eb[i];
    --rem[a];
    --rem[b];
    if (h > target[a] || h > target[b]) return CUDART_INF;
    target[a] -= h;
    target[b] -= h;
    if (!(target[a] <= 2 * rem[a] && target[b] <= 2 * rem[b])) return CUDART_INF;
    halves[i] = h;
    hh[i] = h;
    cst[i + 1] = dadd(cst[i], dmul(dmul(0.5, (double)h), z.c[i]));  // cost + 0.5*h*c
  }
  double best_cost = CUDART_INF;
  enum { ENTER, LOOP, RETURN };
  int i = depth, state = ENTER;
  for (;;) {
    if (state == ENTER) {
      if (cst[i] >= best_cost) {
        state = RETURN;
      } else if (i == mc) {
        best_cost = cst[i];
        for (int k = 0; k < mc; ++k) best[k] = halves[k];
        state = RETURN;
      } else {
        --rem[z.ea[i]];
        --rem[z.eb[i]];
        hh[i] = 0;
        state = LOOP;
      }
    }
    if (state == LOOP) {
      bool descend = false;
      const int a = z.ea[i], b = z.eb[i];
      while (hh[i] <= 2) {
        const int h = hh[i];
        if (h > target[a] || h > target[b]) { hh[i] = 3; break; }
        target[a] -= h;
        target[b] -= h;
        if (target[a] <= 2 * rem[a] && target[b] <= 2 * rem[b]) {
          halves[i] = h;
          cst[i + 1] = dadd(cst[i], dmul(dmul(0.5, (double)h), z.c[i]));  // cost + 0.5*h*c
          descend = true;
          break;
        }
        target[a] += h;
        target[b] += h;
        ++hh[i];
      }
      if (descend) { ++i; state = ENTER; continue; }
      ++rem[a];
      ++rem[b];
      state = RETURN;
    }
    // RETURN to the caller frame (never above the forced prefix)
    if (i == depth) break;
    --i;
    target[z.ea[i]] += hh[i];
    target[z.eb[i]] += hh[i];
    ++hh[i];
    state = LOOP;
  }
  return best_cost;
}

// The whole tree on one thread (k_one_component, the solve_zero_component entry point).
__device__ bool solve_component(const int32_t* comp, int mc, const int32_t* __restrict__ eu,
                                const int32_t* __restrict__ ev, const double* __restrict__ cost,
                                const int32_t* __restrict__ residual, double* __restrict__ x,
                                bool comp_is_sorted_keys, const uint64_t* keys, int ebits) {
  ZeroComponent z;
  component_setup(z, comp, mc, eu, ev, cost, residual, comp_is_sorted_keys, keys, ebits);
  int best[kMaxComponentEdges];
  if (!(component_search(z, 0, 0, best) < CUDART_INF)) return false;  // !isfinite(best_cost)
  for (int k = 0; k < mc; ++k) x[z.ce[k]] = 0.5 * best[k];
  return true;
}

// One warp per zero component: the search tree is split at its first 3 edges into 27 subtrees,
// one per lane, and the lanes' (cost, prefix) minimum is the sequential search's answer
// (see component_search). The exhaustive search of the largest component set this kernel's time
// on one thread (130 us at 100k).
constexpr int kSplitDepth = 3;
__global__ void k_components(int64_t ncomp, int64_t z, const int32_t* __restrict__ heads,
                             const uint64_t* __restrict__ keys, const int32_t* __restrict__ eu,
                             const int32_t* __restrict__ ev, const double* __restrict__ cost,
                             const int32_t* __restrict__ residual, double* __restrict__ x, int ebits,
                             unsigned long long* __restrict__ fail) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncomp) return;  // warp-uniform
  const int64_t lo = heads[c], hi = c + 1 < ncomp ? heads[c + 1] : z;
  const int64_t mc = hi - lo;
  if (mc > kMaxComponentEdges) {  // primal.cpp:210-214
    if (lane == 0) atomicMin(fail, ((unsigned long long)c << 32) | (unsigned long long)mc);
    return;
  }
  ZeroComponent zc;
  component_setup(zc, nullptr, (int)mc, eu, ev, cost, residual, true, keys + lo, ebits);
  const int depth = mc < kSplitDepth ? (int)mc : kSplitDepth;
  const int nprefix = depth == 3 ? 27 : depth == 2 ? 9 : depth == 1 ? 3 : 1;
  int best[kMaxComponentEdges];
  double bc = CUDART_INF;
  int bp = 0x7fffffff;
  if (lane < nprefix) {
    bc = component_search(zc, depth, lane, best);
    bp = lane;
  }
  // lexicographic (cost, prefix) minimum over the lanes; NaN costs never win (as in the DFS)
  double wc = bc;
  int wp = bc < CUDART_INF ? bp : 0x7fffffff;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, wc, off);
    const int op = __shfl_xor_sync(0xffffffffu, wp, off);
    if (oc < wc || (oc == wc && op < wp)) { wc = oc; wp = op; }
  }
  if (!(wc < CUDART_INF)) {
    if (lane == 0) atomicMin(fail, ((unsigned long long)c << 32) | (unsigned long long)(0x80000000u | (unsigned)mc));
    return;
  }
  if (lane == wp)
    for (int k = 0; k < mc; ++k) x[zc.ce[k]] = 0.5 * best[k];
}

__global__ void k_one_component(int mc, const int32_t* __restrict__ comp, const int32_t* __restrict__ eu,
                                const int32_t* __restrict__ ev, const double* __restrict__ cost,
                                const int32_t* __restrict__ residual, double* __restrict__ x,
                                int* __restrict__ ok) {
  *ok = solve_component(comp, mc, eu, ev, cost, residual, x, false, nullptr, 32) ? 1 : 0;
}

__global__ void k_products(int64_t m, const double* __restrict__ cost, const double* __restrict__ x,
                           double* __restrict__ prod) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  prod[e] = dmul(cost[e], x[e]);
}

__global__ void k_node_sums(int n, const int32_t* __restrict__ perm, const int32_t* __restrict__ deg,
                            const int64_t* __restrict__ sptr, const int32_t* __restrict__ seid,
                            const double* __restrict__ x, double* __restrict__ sums,
                            uint8_t* __restrict__ bad) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int p = perm[v];
  const int64_t base = sptr[p >> 5] + (p & 31);
  double s = 0.0;
  for (int j = 0; j < deg[p]; ++j) s = dadd(s, x[seid[base + (int64_t)j * 32]]);
  sums[v] = s;
  bad[v] = s != 2.0;
}

__global__ void k_value_check(int64_t m, const double* __restrict__ x, uint8_t* __restrict__ bad) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const double v = x[e];
  bad[e] = v != 0.0 && v != 0.5 && v != 1.0;
}

// certification counts (no lists): per-node sum != 2.0 (primal.cpp:249-258) and values outside
// {0, 1/2, 1} (primal.cpp:259-266), warp-aggregated atomics
__global__ void k_certify_counts(int n, int64_t m, const int32_t* __restrict__ perm, const int32_t* __restrict__ deg,
                                 const int64_t* __restrict__ sptr, const int32_t* __restrict__ seid,
                                 const double* __restrict__ x, unsigned long long* __restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool nb = false, vb = false;
  if (i < n) {
    const int p = perm[i];
    const int64_t base = sptr[p >> 5] + (p & 31);
    double sum = 0.0;
    for (int j = 0; j < deg[p]; ++j) sum = dadd(sum, x[seid[base + (int64_t)j * 32]]);
    nb = sum != 2.0;
  }
  if (i < m) {
    const double v = x[i];
    vb = v != 0.0 && v != 0.5 && v != 1.0;
  }
  const unsigned bn = __ballot_sync(0xffffffffu, nb), bv = __ballot_sync(0xffffffffu, vb);
  if ((threadIdx.x & 31) == 0) {
    if (bn) atomicAdd(counts, (unsigned long long)__popc(bn));
    if (bv) atomicAdd(counts + 1, (unsigned long long)__popc(bv));
  }
}

template <class T>
static int64_t select_flagged(const T* in, const uint8_t* flags, T* out, int64_t count, cudaStream_t s) {
  DBuf<int64_t> nsel(1, s);
  size_t tmp = 0;
  F2M_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, in, flags, out, nsel.get(), count, s));
  DBuf<char> tb(tmp, s);
  F2M_CUDA(cub::DeviceSelect::Flagged(tb.get(), tmp, in, flags, out, nsel.get(), count, s));
  launched("select_flagged");
  int64_t* ps = pinned_scratch();  // page-locked: a pageable destination would stage the copy
  F2M_CUDA(cudaMemcpyAsync(ps + 12, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  return ps[12];
}

void extract_device(const f2m_graph& g, const double* d_lam_pos, double tol, double* d_x) {
  if (!(tol > 0.0)) throw Error(F2M_E_ARGUMENT, "classify_edges: tol must be > 0");
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int n = t.n;
  const int64_t m = t.m;
  DBuf<uint8_t> label(std::max<int64_t>(m, 1), s), zflag(std::max<int64_t>(m, 1), s);
  DBuf<int32_t> negd(std::max(n, 1), s), zerod(std::max(n, 1), s), residual(std::max(n, 1), s);
  if (n > 0) {
    F2M_CUDA(cudaMemsetAsync(negd.get(), 0, sizeof(int32_t) * n, s));
    F2M_CUDA(cudaMemsetAsync(zerod.get(), 0, sizeof(int32_t) * n, s));
  }
  if (m > 0) {
    k_classify<<<grid_for(m, 256), 256, 0, s>>>(m, t.eu.get(), t.ev.get(), g.cost.get(), t.perm.get(), d_lam_pos,
                                               tol, label.get(), negd.get(), zerod.get(), d_x, zflag.get());
    launched("classify");
  }
  DBuf<unsigned long long> first(1, s);
  F2M_CUDA(cudaMemsetAsync(first.get(), 0xff, sizeof(unsigned long long), s));
  if (n > 0) {
    k_check_nodes<<<grid_for(n, 256), 256, 0, s>>>(n, negd.get(), zerod.get(), residual.get(), first.get());
    launched("check_nodes");
  }
  // the node check's verdict comes back with the next synchronisation (the zero-band selection)
  unsigned long long* hfirst = reinterpret_cast<unsigned long long*>(pinned_scratch() + 13);
  F2M_CUDA(cudaMemcpyAsync(hfirst, first.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  auto check_nodes = [&] {  // primal.cpp:155-175 order: node degrees before the zero components
    if (*hfirst == ~0ULL) return;
    const int v = (int)(*hfirst / 2);
    int nd = 0;
    F2M_CUDA(cudaMemcpy(&nd, negd.get() + v, sizeof(int), cudaMemcpyDeviceToHost));
    if (*hfirst % 2 == 0)
      throw Error(F2M_E_DEGENERATE, "node " + std::to_string(v) + " has " + std::to_string(nd) + " tight edges (> 2)");
    throw Error(F2M_E_DEGENERATE, "node " + std::to_string(v) + " needs " + std::to_string(2 - nd) +
                                      " more units but has no zero-band edge");
  };
  if (m == 0) {
    F2M_CUDA(cudaStreamSynchronize(s));
    check_nodes();
    return;
  }
  // zero-band edges, ascending
  DBuf<int32_t> eids(m, s), zedges(m, s);
  k_iota_n<<<grid_for(m, 256), 256, 0, s>>>((int)m, eids.get());
  launched("iota");
  const int64_t z = select_flagged<int32_t>(eids.get(), zflag.get(), zedges.get(), m, s);
  check_nodes();
  if (z == 0) return;
  DBuf<int> parent(n, s);
  k_iota_n<<<grid_for(n, 256), 256, 0, s>>>(n, parent.get());
  launched("iota");
  k_union<<<grid_for(z, 256), 256, 0, s>>>(z, zedges.get(), t.eu.get(), t.ev.get(), parent.get());
  launched("union_find");
  DBuf<uint64_t> k0(z, s), k1(z, s);
  const int ebits = std::max(bit_width(m - 1), 1), key_bits = ebits + std::max(bit_width(n - 1), 1);
  k_comp_keys<<<grid_for(z, 256), 256, 0, s>>>(z, zedges.get(), t.eu.get(), parent.get(), ebits, k0.get());
  launched("comp_keys");
  {
    size_t tmp = 0;
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0.get(), k1.get(), z, 0, key_bits, s));
    DBuf<char> tb(tmp, s);
    F2M_CUDA(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k0.get(), k1.get(), z, 0, key_bits, s));
    launched("sort_components");
  }
  DBuf<uint8_t> head(z, s);
  k_heads<<<grid_for(z, 256), 256, 0, s>>>(z, k1.get(), ebits, head.get());
  launched("heads");
  DBuf<int32_t> zi(z, s), heads(z, s);
  k_iota_n<<<grid_for(z, 256), 256, 0, s>>>((int)z, zi.get());
  launched("iota");
  const int64_t ncomp = select_flagged<int32_t>(zi.get(), head.get(), heads.get(), z, s);
  DBuf<unsigned long long> fail(1, s);
  F2M_CUDA(cudaMemsetAsync(fail.get(), 0xff, sizeof(unsigned long long), s));
  k_components<<<grid_for(ncomp * 32, 128), 128, 0, s>>>(ncomp, z, heads.get(), k1.get(), t.eu.get(), t.ev.get(),
                                                        g.cost.get(), residual.get(), d_x, ebits, fail.get());
  launched("zero_components");
  unsigned long long* hfp = reinterpret_cast<unsigned long long*>(pinned_scratch() + 14);
  F2M_CUDA(cudaMemcpyAsync(hfp, fail.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  const unsigned long long hf = *hfp;
  if (hf != ~0ULL) {
    const unsigned low = (unsigned)(hf & 0xffffffffu);
    const unsigned mc = low & 0x7fffffffu;
    if (low & 0x80000000u)
      throw Error(F2M_E_DEGENERATE, "no feasible {0, 1/2, 1} completion for a zero component of " +
                                        std::to_string(mc) + " edges");
    throw Error(F2M_E_DEGENERATE, "zero component with " + std::to_string(mc) +
                                      " edges exceeds the exhaustive-search cap of " +
                                      std::to_string(kMaxComponentEdges));
  }
}

double objective_device(const f2m_graph& g, const double* d_x) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int64_t m = t.m;
  if (m == 0) return 0.0;
  DBuf<double> prod(m, s), out(1, s);
  k_products<<<grid_for(m, 256), 256, 0, s>>>(m, g.cost.get(), d_x, prod.get());
  launched("products");
  seq_sums_device(prod.get(), m, m, out.get(), s);  // the reference's left-to-right chain, exactly
  double h = 0.0;
  F2M_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  return h;
}

void verify_device(const f2m_graph& g, const double* d_x, double objective, const double* d_lam_pos,
                   f2m_verification& rep, int32_t* h_nodes, double* h_sums, int32_t* h_vals,
                   int64_t capacity, const double* dual_known) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int n = t.n;
  const int64_t m = t.m;
  int64_t nbad = 0, vbad = 0;
  if (n > 0) {
    DBuf<double> sums(n, s), bsums(n, s);
    DBuf<uint8_t> bad(n, s);
    DBuf<int32_t> ids(n, s), bids(n, s);
    k_node_sums<<<grid_for(n, 256), 256, 0, s>>>(n, t.perm.get(), t.deg.get(), t.sptr.get(), t.seid.get(), d_x,
                                                sums.get(), bad.get());
    launched("node_sums");
    k_iota_n<<<grid_for(n, 256), 256, 0, s>>>(n, ids.get());
    launched("iota");
    nbad = select_flagged<int32_t>(ids.get(), bad.get(), bids.get(), n, s);
    if (nbad > 0 && (h_nodes || h_sums)) {
      select_flagged<double>(sums.get(), bad.get(), bsums.get(), n, s);
      const int64_t k = std::min(nbad, capacity);
      if (h_nodes && k) F2M_CUDA(cudaMemcpy(h_nodes, bids.get(), sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
      if (h_sums && k) F2M_CUDA(cudaMemcpy(h_sums, bsums.get(), sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
  }
  if (m > 0) {
    DBuf<uint8_t> bad(m, s);
    DBuf<int32_t> ids(m, s), bids(m, s);
    k_value_check<<<grid_for(m, 256), 256, 0, s>>>(m, d_x, bad.get());
    launched("value_check");
    k_iota_n<<<grid_for(m, 256), 256, 0, s>>>((int)m, ids.get());
    launched("iota");
    vbad = select_flagged<int32_t>(ids.get(), bad.get(), bids.get(), m, s);
    const int64_t k = std::min(vbad, capacity);
    if (h_vals && k) F2M_CUDA(cudaMemcpy(h_vals, bids.get(), sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
  }
  rep.violated_count = nbad;
  rep.value_violation_count = vbad;
  rep.feasible = nbad == 0 && vbad == 0;
  // dual_objective(graph, state) (primal.cpp:274); solve_duals already computed it for the same
  // graph, lambda and b when the caller passes it in
  rep.duality_gap = objective - (dual_known ? *dual_known : dual_objective_device(g, d_lam_pos, 2));
}

void certify_device(const f2m_graph& g, const double* d_x, double dual, double& objective, f2m_verification& rep) {
  const Topology& t = *g.topo;
  cudaStream_t s = t.stream;
  const int n = t.n;
  const int64_t m = t.m;
  DBuf<unsigned long long> counts(2, s);
  DBuf<double> obj(1, s);
  F2M_CUDA(cudaMemsetAsync(counts.get(), 0, 2 * sizeof(unsigned long long), s));
  F2M_CUDA(cudaMemsetAsync(obj.get(), 0, sizeof(double), s));
  if (m > 0) {
    DBuf<double> prod(m, s);
    k_products<<<grid_for(m, 256), 256, 0, s>>>(m, g.cost.get(), d_x, prod.get());
    launched("products");
    seq_sums_device(prod.get(), m, m, obj.get(), s);  // the reference's left-to-right chain, exactly
  }
  const int64_t items = std::max<int64_t>(n, m);
  if (items > 0) {
    k_certify_counts<<<grid_for(items, 256), 256, 0, s>>>(n, m, t.perm.get(), t.deg.get(), t.sptr.get(),
                                                         t.seid.get(), d_x, counts.get());
    launched("certify_counts");
  }
  int64_t* ps = pinned_scratch();
  F2M_CUDA(cudaMemcpyAsync(ps + 26, obj.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaMemcpyAsync(ps + 27, counts.get(), 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  F2M_CUDA(cudaStreamSynchronize(s));
  std::memcpy(&objective, ps + 26, sizeof(double));
  rep.violated_count = ps[27];
  rep.value_violation_count = ps[28];
  rep.feasible = ps[27] == 0 && ps[28] == 0;
  rep.duality_gap = objective - dual;  // primal.cpp:274
}

}  // namespace f2mgpu

using namespace f2mgpu;

extern "C" int f2m_classify_edges(const f2m_graph* g, const double* lambda, double tol, uint8_t* label) {
  return guard([&] {
    if (!(tol > 0.0)) throw Error(F2M_E_ARGUMENT, "classify_edges: tol must be > 0");
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    DBuf<double> lam(std::max(t.n, 1), s);
    upload_lambda(*g, lambda, lam.get());
    DBuf<uint8_t> d_label(std::max<int64_t>(t.m, 1), s);
    if (t.m > 0) {
      k_classify<<<grid_for(t.m, 256), 256, 0, s>>>(t.m, t.eu.get(), t.ev.get(), g->cost.get(), t.perm.get(),
                                                    lam.get(), tol, d_label.get(), nullptr, nullptr, nullptr,
                                                    nullptr);
      launched("classify");
      F2M_CUDA(cudaMemcpyAsync(label, d_label.get(), t.m, cudaMemcpyDeviceToHost, s));
    }
    F2M_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int f2m_extract_primal(const f2m_graph* g, const double* lambda, double tol, double* x,
                                  double* objective) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    DBuf<double> lam(std::max(t.n, 1), s), dx(std::max<int64_t>(t.m, 1), s);
    upload_lambda(*g, lambda, lam.get());
    extract_device(*g, lam.get(), tol, dx.get());
    *objective = objective_device(*g, dx.get());
    if (t.m > 0) F2M_CUDA(cudaMemcpyAsync(x, dx.get(), sizeof(double) * t.m, cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int f2m_solve_zero_component(const f2m_graph* g, const int32_t* component_edges, int count,
                                        const int32_t* residual, double* values, int* feasible) {
  return guard([&] {
    const Topology& t = *g->topo;
    if (count < 0 || count > kMaxComponentEdges)
      throw Error(F2M_E_ARGUMENT, "solve_zero_component: component size must be in [0, 20]");
    for (int i = 0; i < count; ++i)
      if (component_edges[i] < 0 || component_edges[i] >= t.m) throw Error(F2M_E_INDEX, "edge id out of range");
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    if (count == 0) { *feasible = 1; return; }
    DBuf<int32_t> comp(count, s), res(std::max(t.n, 1), s);
    DBuf<double> dx(std::max<int64_t>(t.m, 1), s);
    DBuf<int> ok(1, s);
    F2M_CUDA(cudaMemcpyAsync(comp.get(), component_edges, sizeof(int32_t) * count, cudaMemcpyHostToDevice, s));
    if (t.n > 0) F2M_CUDA(cudaMemcpyAsync(res.get(), residual, sizeof(int32_t) * t.n, cudaMemcpyHostToDevice, s));
    k_one_component<<<1, 1, 0, s>>>(count, comp.get(), t.eu.get(), t.ev.get(), g->cost.get(), res.get(), dx.get(),
                                    ok.get());
    launched("one_component");
    int hok = 0;
    F2M_CUDA(cudaMemcpyAsync(&hok, ok.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    std::vector<double> hx(t.m);
    if (t.m > 0) F2M_CUDA(cudaMemcpyAsync(hx.data(), dx.get(), sizeof(double) * t.m, cudaMemcpyDeviceToHost, s));
    F2M_CUDA(cudaStreamSynchronize(s));
    *feasible = hok;
    if (hok)
      for (int i = 0; i < count; ++i) values[i] = hx[component_edges[i]];
  });
}

extern "C" int f2m_verify_solution(const f2m_graph* g, const double* x, double objective, const double* lambda,
                                   f2m_verification* report, int32_t* violated_nodes, double* violated_sums,
                                   int32_t* value_violations, int64_t capacity) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t s = t.stream;
    DBuf<double> lam(std::max(t.n, 1), s), dx(std::max<int64_t>(t.m, 1), s);
    upload_lambda(*g, lambda, lam.get());
    if (t.m > 0) F2M_CUDA(cudaMemcpyAsync(dx.get(), x, sizeof(double) * t.m, cudaMemcpyHostToDevice, s));
    verify_device(*g, dx.get(), objective, lam.get(), *report, violated_nodes, violated_sums, value_violations,
                  capacity);
  });
}

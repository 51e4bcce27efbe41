// shard.cu — node-sharded multi-GPU GDP: the per-rank sweep kernel and the
// position-order helpers the host driver (paper_2011_08170_b200/sharded.py) needs.
//
// Rank r of `world` owns the contiguous spatial positions [r*stride, min(n, (r+1)*stride)),
// stride = ceil(n / world). The k-NN grid's Morton order makes each range a compact patch of the
// plane, so most of a shard's neighbour reads stay inside its own range. A sweep reads the full
// multiplier vector of the previous sweep (the NCCL all-gather of all shards) and writes only the
// owned entries, which is the reference's frozen-snapshot Jacobi sweep (dual.cpp:129-167)
// restricted to a row range: the result is bit-identical for every world size.
//
//  k_shard_sweep<B>  one launch per sweep, one thread per owned row, SELL-32 slot loads
//                    (coalesced across the warp), neighbour multipliers gathered from the
//                    (L2-resident) full vector; block max |delta| -> one 64-bit atomicMax on the
//                    IEEE bits (|delta| >= 0, so bit order == value order).
#include "internal.cuh"

struct f2m_shard {
  std::shared_ptr<f2mgpu::Topology> topo;
  const f2m_graph* g = nullptr;  // costs (scost) of the graph the shard was cut from
  int rank = 0, world = 1;
  int begin = 0, end = 0, stride = 0;
  int64_t slots = 0;
};

namespace f2mgpu {

constexpr int kShardThreads = 256;

template <int B>
__global__ void __launch_bounds__(kShardThreads) k_shard_sweep(
    int begin, int end, int stride, const int64_t* __restrict__ sptr, const int32_t* __restrict__ swidth,
    const int32_t* __restrict__ scol, const double* __restrict__ scost, const double* __restrict__ lam,
    double* __restrict__ out, double eta, int update, unsigned long long* __restrict__ max_bits) {
  __shared__ unsigned long long wmax[kShardThreads / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // owned position index (0..stride)
  const int p = begin + i;
  double ad = 0.0;
  if (i < stride) {
    if (p < end) {
      const int sl = p >> 5;
      const int64_t base = sptr[sl] + (p & 31);
      const int w = swidth[sl];
      const double lv = lam[p];
      double s[B + 1];
#pragma unroll
      for (int k = 0; k <= B; ++k) s[k] = CUDART_INF;
      // batches of 8 slots: 16 streaming loads (evict-first, so the L2 keeps the gathered
      // multipliers) and then 8 independent gathers in flight per thread
      for (int j = 0; j < w; j += 8) {
        int q[8];
        double c[8], l[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = j + u < w;
          const int64_t idx = base + (int64_t)(ok ? j + u : 0) * 32;
          q[u] = ok ? __ldcs(scol + idx) : p;
          c[u] = ok ? __ldcs(scost + idx) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) l[u] = lam[q[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j + u < w) topk_bubble<B>(s, dsub(dsub(c[u], lv), l[u]));
      }
      // delta_for (dual.cpp:63-68), lambda += eta * delta (dual.cpp:157-161)
      const double d = update ? dmul(0.5, dsub(s[B - 1], s[B])) : dmul(0.5, dadd(s[B - 1], s[B]));
      out[i] = dadd(lv, dmul(eta, d));
      ad = fabs(d);
      if (ad != ad) ad = 0.0;  // std::max(local_max, NaN) keeps local_max (dual.cpp:149)
    } else {
      out[i] = 0.0;  // padding
    }
  }
  const unsigned long long v = (unsigned long long)__double_as_longlong(ad);
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32) == hi ? (unsigned)v : 0u);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = ((unsigned long long)hi << 32) | lo;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int k = 0; k < kShardThreads / 32; ++k) m = wmax[k] > m ? wmax[k] : m;
    if (m) atomicMax(max_bits, m);
  }
}

template <int B>
static void launch_shard(const f2m_shard& sh, const f2m_engine_config& cfg, const double* lam, double* out,
                         unsigned long long* max_bits, cudaStream_t st) {
  const Topology& t = *sh.topo;
  const int blocks = (sh.stride + kShardThreads - 1) / kShardThreads;
  if (blocks == 0) return;
  k_shard_sweep<B><<<blocks, kShardThreads, 0, st>>>(sh.begin, sh.end, sh.stride, t.sptr.get(), t.swidth.get(),
                                                    t.scol.get(), sh.g->scost.get(), lam, out, cfg.eta, cfg.update,
                                                    max_bits);
  launched("shard_sweep");
}

__global__ void k_perm_gather(int n, const double* __restrict__ src, const int32_t* __restrict__ idx,
                              double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_pack(int64_t count, const double* __restrict__ src, const int32_t* __restrict__ idx,
                       double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < count) dst[i] = src[idx[i]];
}

__global__ void k_unpack(int64_t count, const double* __restrict__ src, const int32_t* __restrict__ idx,
                         double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < count) dst[idx[i]] = src[i];
}

}  // namespace f2mgpu

using namespace f2mgpu;

extern "C" int f2m_shard_create(const f2m_graph* g, int rank, int world, f2m_shard** out) {
  return guard([&] {
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) throw Error(F2M_E_ARGUMENT, "shard: need 0 <= rank < world");
    const Topology& t = *g->topo;
    auto sh = std::make_unique<f2m_shard>();
    sh->topo = g->topo;
    sh->g = g;
    sh->rank = rank;
    sh->world = world;
    sh->stride = (t.n + world - 1) / world;
    sh->begin = std::min(t.n, rank * sh->stride);
    sh->end = std::min(t.n, (rank + 1) * sh->stride);
    if (sh->end > sh->begin) {
      int64_t lo = 0, hi = 0;
      const int s0 = sh->begin >> 5, s1 = (sh->end - 1) >> 5;
      F2M_CUDA(cudaSetDevice(t.dev));
      F2M_CUDA(cudaMemcpy(&lo, t.sptr.get() + s0, sizeof(int64_t), cudaMemcpyDeviceToHost));
      F2M_CUDA(cudaMemcpy(&hi, t.sptr.get() + s1 + 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
      sh->slots = hi - lo;
    }
    *out = sh.release();
  });
}

extern "C" void f2m_shard_destroy(f2m_shard* s) { delete s; }

extern "C" int f2m_shard_get_info(const f2m_shard* s, f2m_shard_info* out) {
  return guard([&] {
    out->n = s->topo->n;
    out->rank = s->rank;
    out->world = s->world;
    out->begin = s->begin;
    out->end = s->end;
    out->stride = s->stride;
    out->slots = s->slots;
  });
}

extern "C" int f2m_shard_sweep(const f2m_shard* s, const f2m_engine_config* cfg, const double* d_lam_full,
                               double* d_lam_shard, unsigned long long* d_max_bits, void* stream) {
  return guard([&] {
    validate_engine(*cfg);
    const Topology& t = *s->topo;
    if (t.n > 0 && t.min_deg <= cfg->b)
      throw Error(F2M_E_DEGREE, "node has degree " + std::to_string(t.min_deg) + " <= b = " + std::to_string(cfg->b));
    F2M_CUDA(cudaSetDevice(t.dev));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (cfg->b) {
      case 1: launch_shard<1>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 2: launch_shard<2>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 3: launch_shard<3>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 4: launch_shard<4>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 5: launch_shard<5>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 6: launch_shard<6>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      case 7: launch_shard<7>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
      default: launch_shard<8>(*s, *cfg, d_lam_full, d_lam_shard, d_max_bits, st); break;
    }
  });
}

extern "C" int f2m_initial_state_positions(const f2m_graph* g, const f2m_engine_config* cfg, double* d_lam_pos,
                                           void* stream) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (cfg->b < 1 || cfg->b > kMaxB) throw Error(F2M_E_ARGUMENT, "make_initial_state: b out of range");
    // the caller's pending work on d_lam_pos is ordered before the init on the graph stream
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaEvent_t ev;
    F2M_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    F2M_CUDA(cudaEventRecord(ev, st));
    F2M_CUDA(cudaStreamWaitEvent(t.stream, ev, 0));
    initial_state_device(*g, *cfg, d_lam_pos);  // synchronises the graph stream
    cudaEventDestroy(ev);
  });
}

extern "C" int f2m_positions_to_ids(const f2m_graph* g, const double* d_pos, double* d_ids, void* stream) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.n == 0) return;
    // ids[v] = pos[perm[v]]
    k_perm_gather<<<grid_for(t.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(t.n, d_pos, t.perm.get(), d_ids);
    launched("positions_to_ids");
  });
}

extern "C" int f2m_ids_to_positions(const f2m_graph* g, const double* d_ids, double* d_pos, void* stream) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.n == 0) return;
    // pos[p] = ids[iperm[p]]
    k_perm_gather<<<grid_for(t.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(t.n, d_ids, t.iperm.get(), d_pos);
    launched("ids_to_positions");
  });
}

extern "C" int f2m_graph_positions(const f2m_graph* g, int32_t* position) {
  return guard([&] {
    const Topology& t = *g->topo;
    F2M_CUDA(cudaSetDevice(t.dev));
    if (t.n > 0) F2M_CUDA(cudaMemcpy(position, t.perm.get(), sizeof(int32_t) * t.n, cudaMemcpyDeviceToHost));
  });
}

extern "C" int f2m_gather_f64(const double* d_src, const int32_t* d_idx, double* d_dst, int64_t count, void* stream) {
  return guard([&] {
    if (count <= 0) return;
    k_pack<<<grid_for(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(count, d_src, d_idx, d_dst);
    launched("halo_pack");
  });
}

extern "C" int f2m_scatter_f64(const double* d_src, const int32_t* d_idx, double* d_dst, int64_t count, void* stream) {
  return guard([&] {
    if (count <= 0) return;
    k_unpack<<<grid_for(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(count, d_src, d_idx, d_dst);
    launched("halo_unpack");
  });
}

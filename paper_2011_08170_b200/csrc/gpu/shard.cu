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

// One Jacobi row update of position p (dual.cpp:129-167 for one node): top-(B+1) of
// (c - lambda_p) - lambda_q over the row's SELL slots, midpoint / difference delta. Returns the
// new multiplier; |delta| in ad (NaN skipped like std::max(local_max, NaN), dual.cpp:149).
template <int B>
__device__ __forceinline__ double shard_row(int p, const int64_t* __restrict__ sptr, const int32_t* __restrict__ swidth,
                                            const int32_t* __restrict__ scol, const double* __restrict__ scost,
                                            const double* lam, double eta, int update, double& ad) {
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
  ad = fabs(d);
  if (ad != ad) ad = 0.0;
  return dadd(lv, dmul(eta, d));
}

// block max of non-negative doubles through their IEEE bits -> one atomicMax per block
__device__ __forceinline__ void block_max_bits(double ad, unsigned long long* smem_w, unsigned long long* target) {
  const unsigned long long v = (unsigned long long)__double_as_longlong(ad);
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32) == hi ? (unsigned)v : 0u);
  if ((threadIdx.x & 31) == 0) smem_w[threadIdx.x >> 5] = ((unsigned long long)hi << 32) | lo;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = smem_w[k] > m ? smem_w[k] : m;
    if (m) atomicMax(target, m);
  }
}

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
    if (p < end) out[i] = shard_row<B>(p, sptr, swidth, scol, scost, lam, eta, update, ad);
    else out[i] = 0.0;  // padding
  }
  block_max_bits(ad, wmax, max_bits);
}

// ---------------------------------------------------------------- fused peer-memory solve
// SURVEY §8(e) "faster fused variant": one persistent kernel per rank runs ALL sweeps; the halo
// multipliers go straight into the reader's receive buffer with device-initiated stores (peer
// memory over NVLink, LL words {tag:32 | half:32}, system scope), every rank stores its sweep
// max |delta| into every rank's board, and every rank takes the same stop decision from the same
// maxima. No host round trip, no NCCL launch per sweep. Per sweep: [receive halo s] barrier
// [rows] barrier [send halo s+1, publish max; every CTA decides from the boards]. Ranks stay within one sweep of
// each other (each waits for all maxima of sweep s), so two receive-buffer parities and a
// 4-slot board ring never overwrite unread words.
struct P2PCtl {
  unsigned bar;
  int error;
  int decision;  // 0 running, 1 converged, 2 sweep budget spent
  int sweeps;
  int out_buffer;
  int pad;
  double final_max;
  unsigned long long maxbits[4];
};

struct P2PArgs {
  int begin, end;
  const int64_t* __restrict__ sptr;
  const int32_t* __restrict__ swidth;
  const int32_t* __restrict__ scol;
  const double* __restrict__ scost;
  double* lam_a;  // full-length position-order vectors; lam_a holds lambda_0 on entry
  double* lam_b;
  const int32_t* __restrict__ recv_pos;
  int64_t n_recv;
  unsigned long long* recv_buf;  // 2 parities x n_recv LL pairs (written by the owners)
  const int32_t* __restrict__ send_pos;
  const int32_t* __restrict__ send_peer;
  const int32_t* __restrict__ send_dst;
  int64_t n_send;
  unsigned long long* const* peer_recv;  // [world] receive buffers of every rank
  const int64_t* peer_nrecv;             // [world]
  unsigned long long* board;             // 4 x world LL pairs (written by every rank)
  unsigned long long* const* peer_board; // [world]
  int world, rank;
  double eta;
  int update;
  double threshold;
  int max_sweeps;
  P2PCtl* ctl;
};

constexpr uint64_t kP2PWatchdogNs = 20ull * 1000000000ull;

__device__ __forceinline__ void st_ll_sys(unsigned long long* p, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long hi = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)),
               "l"(hi | (b >> 32))
               : "memory");
}
__device__ __forceinline__ bool ld_ll_sys(const unsigned long long* p, unsigned tag, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  if ((unsigned)(w0 >> 32) != tag || (unsigned)(w1 >> 32) != tag) return false;
  v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return true;
}
// poll an LL pair until it carries `tag`; false (and ctl->error) on the watchdog
__device__ __forceinline__ bool poll_ll_sys(const unsigned long long* p, unsigned tag, double& v, P2PCtl* ctl) {
  const uint64_t t0 = globaltimer_ns();
  int it = 0;
  while (!ld_ll_sys(p, tag, v)) {
    if ((++it & 255) == 0 && (ld_relaxed(&ctl->error) || globaltimer_ns() - t0 > kP2PWatchdogNs)) {
      atomicExch(&ctl->error, 1);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ void p2p_barrier(P2PCtl* ctl, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&ctl->bar, 1u);
    const uint64_t t0 = globaltimer_ns();
    while (ld_relaxed_u32(&ctl->bar) < target) {
      if (globaltimer_ns() - t0 > kP2PWatchdogNs) {
        atomicExch(&ctl->error, 1);
        break;
      }
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kP2PThreads = 1024;  // one CTA per SM: 148 arrivals per grid barrier

template <int B>
__global__ void __launch_bounds__(kP2PThreads, 1) k_p2p_solve(P2PArgs a) {
  __shared__ unsigned long long wmax[kP2PThreads / 32];
  P2PCtl* ctl = a.ctl;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  unsigned target = 0;
  double* cur = a.lam_a;
  double* nxt = a.lam_b;
  for (int s = 0;; ++s) {
    if (s > 0) {  // halo of sweep s: written by its owners with tag s into parity s & 1
      const unsigned long long* rb = a.recv_buf + (size_t)(s & 1) * a.n_recv * 2;
      for (int64_t i = gtid; i < a.n_recv; i += gsize) {
        double v = 0.0;
        if (poll_ll_sys(rb + 2 * i, (unsigned)s, v, ctl)) cur[a.recv_pos[i]] = v;
      }
      p2p_barrier(ctl, target);
    }
    double ad_max = 0.0;
    for (int64_t i = gtid; i < a.end - a.begin; i += gsize) {
      const int p = a.begin + (int)i;
      double ad = 0.0;
      nxt[p] = shard_row<B>(p, a.sptr, a.swidth, a.scol, a.scost, cur, a.eta, a.update, ad);
      ad_max = ad_max < ad ? ad : ad_max;
    }
    block_max_bits(ad_max, wmax, &ctl->maxbits[s & 3]);
    p2p_barrier(ctl, target);
    for (int64_t j = gtid; j < a.n_send; j += gsize) {  // halo of sweep s+1 into the readers
      const int q = a.send_peer[j];
      unsigned long long* dst = a.peer_recv[q] + 2 * ((size_t)((s + 1) & 1) * a.peer_nrecv[q] + a.send_dst[j]);
      st_ll_sys(dst, nxt[a.send_pos[j]], (unsigned)s + 1);
    }
    // every CTA takes the stop decision itself from the boards (same maxima -> same decision):
    // no third grid barrier per sweep
    __shared__ int s_dec;
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        const unsigned long long mine = *(volatile unsigned long long*)&ctl->maxbits[s & 3];
        ctl->maxbits[(s + 2) & 3] = 0ull;  // reused two sweeps later, after two more barriers
        for (int q = 0; q < a.world; ++q)
          st_ll_sys(a.peer_board[q] + 2 * ((size_t)(s & 3) * a.world + a.rank),
                    __longlong_as_double((long long)mine), (unsigned)s + 1);
      }
      unsigned long long gm = 0;
      bool ok = true;
      for (int q = 0; q < a.world && ok; ++q) {
        double v = 0.0;
        ok = poll_ll_sys(a.board + 2 * ((size_t)(s & 3) * a.world + q), (unsigned)s + 1, v, ctl);
        const unsigned long long b = (unsigned long long)__double_as_longlong(v);
        gm = b > gm ? b : gm;
      }
      const double gmax = __longlong_as_double((long long)gm);
      // solve_duals (dual.cpp:232-238): converged iff max|delta| <= eps * mean_cost
      int dec = gmax <= a.threshold ? 1 : (s + 1 >= a.max_sweeps ? 2 : 0);
      if (!ok || ld_relaxed(&ctl->error)) dec = 2;
      if (dec && blockIdx.x == 0) {
        ctl->sweeps = s + 1;
        ctl->final_max = gmax;
        ctl->out_buffer = nxt == a.lam_b ? 1 : 0;
        ctl->decision = dec;
      }
      s_dec = dec;
    }
    __syncthreads();
    if (s_dec) break;
    double* t = cur;
    cur = nxt;
    nxt = t;
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

template <int B>
static void launch_p2p(const P2PArgs& a, int ctas, cudaStream_t st) {
  void* args[] = {(void*)&a};
  F2M_CUDA(cudaLaunchCooperativeKernel((const void*)k_p2p_solve<B>, dim3(ctas), dim3(kP2PThreads), args, 0, st));
  launched("p2p_solve");
}

extern "C" size_t f2m_p2p_ctl_bytes(void) { return sizeof(f2mgpu::P2PCtl); }

template <int B>
static int p2p_occupancy() {
  int per_sm = 0;
  F2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p2p_solve<B>, kP2PThreads, 0));
  return per_sm;
}

extern "C" int f2m_p2p_max_ctas(int b) {
  int out = 0;
  const int st = guard([&] {
    int per_sm = 0;
    switch (b) {
      case 1: per_sm = p2p_occupancy<1>(); break;
      case 2: per_sm = p2p_occupancy<2>(); break;
      case 3: per_sm = p2p_occupancy<3>(); break;
      case 4: per_sm = p2p_occupancy<4>(); break;
      case 5: per_sm = p2p_occupancy<5>(); break;
      case 6: per_sm = p2p_occupancy<6>(); break;
      case 7: per_sm = p2p_occupancy<7>(); break;
      default: per_sm = p2p_occupancy<8>(); break;
    }
    out = std::max(1, per_sm) * device_props(current_device()).multiProcessorCount;
  });
  return st == F2M_OK ? out : -st;
}

extern "C" int f2m_p2p_launch(const f2m_shard* sh, const f2m_engine_config* cfg, const f2m_p2p_plan* plan,
                              double* d_lam_a, double* d_lam_b, double threshold, int max_sweeps, int ctas,
                              void* d_ctl, void* stream) {
  return guard([&] {
    validate_engine(*cfg);
    const Topology& t = *sh->topo;
    if (t.n > 0 && t.min_deg <= cfg->b)
      throw Error(F2M_E_DEGREE, "node has degree " + std::to_string(t.min_deg) + " <= b = " + std::to_string(cfg->b));
    if (max_sweeps < 1) throw Error(F2M_E_ARGUMENT, "p2p solve: max_sweeps must be >= 1");
    F2M_CUDA(cudaSetDevice(t.dev));
    P2PArgs a;
    a.begin = sh->begin;
    a.end = sh->end;
    a.sptr = t.sptr.get();
    a.swidth = t.swidth.get();
    a.scol = t.scol.get();
    a.scost = sh->g->scost.get();
    a.lam_a = d_lam_a;
    a.lam_b = d_lam_b;
    a.recv_pos = plan->d_recv_pos;
    a.n_recv = plan->n_recv;
    a.recv_buf = plan->d_recv_buf;
    a.send_pos = plan->d_send_pos;
    a.send_peer = plan->d_send_peer;
    a.send_dst = plan->d_send_dst;
    a.n_send = plan->n_send;
    a.peer_recv = plan->d_peer_recv;
    a.peer_nrecv = plan->d_peer_nrecv;
    a.board = plan->d_board;
    a.peer_board = plan->d_peer_board;
    a.world = sh->world;
    a.rank = sh->rank;
    a.eta = cfg->eta;
    a.update = cfg->update;
    a.threshold = threshold;
    a.max_sweeps = max_sweeps;
    a.ctl = static_cast<P2PCtl*>(d_ctl);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    F2M_CUDA(cudaMemsetAsync(d_ctl, 0, sizeof(P2PCtl), st));
    const int g = std::max(1, ctas);
    switch (cfg->b) {
      case 1: launch_p2p<1>(a, g, st); break;
      case 2: launch_p2p<2>(a, g, st); break;
      case 3: launch_p2p<3>(a, g, st); break;
      case 4: launch_p2p<4>(a, g, st); break;
      case 5: launch_p2p<5>(a, g, st); break;
      case 6: launch_p2p<6>(a, g, st); break;
      case 7: launch_p2p<7>(a, g, st); break;
      default: launch_p2p<8>(a, g, st); break;
    }
  });
}

extern "C" int f2m_p2p_get_result(const void* d_ctl, f2m_p2p_result* out) {
  return guard([&] {
    P2PCtl h;
    F2M_CUDA(cudaMemcpy(&h, d_ctl, sizeof(h), cudaMemcpyDeviceToHost));
    if (h.error) throw Error(F2M_E_TIMEOUT, "p2p solve: a peer did not answer within the watchdog (20 s)");
    out->sweeps = h.sweeps;
    out->converged = h.decision == 1 ? 1 : 0;
    out->out_buffer = h.out_buffer;
    out->final_max_abs_delta = h.final_max;
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

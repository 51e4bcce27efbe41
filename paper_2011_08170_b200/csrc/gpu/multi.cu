// multi.cu — solve_duals (dual.cpp:210-246) on several GPUs from ONE host thread.
//
// The reference's C++ entry point `solve_duals(graph, config)` (dual.hpp:79-81) reaches more than
// one B200 through EngineConfig::num_gpus (f2m_engine_config.num_gpus): no torch.distributed, no
// extra processes. The engine is the partition-resident persistent sweep kernel (k_gdp_sweep5)
// spread over the GPUs exactly as the torch-driven ShardedResident does it (sharded.py), with the
// peer memory coming from CUDA peer access instead of torch symmetric memory:
//   * the graph is replicated onto every GPU and partitioned into world x Gp CTAs (Gp = SMs - 1, or
//     fewer when several ranks share one GPU — the test configuration, f2m_set_gpu_list);
//   * rank r launches partition CTAs [r*Gp, (r+1)*Gp) + its own convergence master on its GPU; every
//     boundary multiplier is stored (st.relaxed.sys, NVLink) into the LL ring of each rank that
//     reads it and every CTA's sweep max into every rank's max ring, so all masters issue the same
//     verdicts with no host work, barrier or collective per sweep;
//   * after the stopping sweep each rank's owned range is copied (peer copy) onto the primary GPU.
// Bit-identical to the one-GPU solve: a Jacobi sweep reads only the frozen multipliers, and the
// convergence verdicts are the same maxima compared with the same threshold.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>

#include "internal.cuh"

namespace f2mgpu {

static std::mutex g_gpu_list_mu;
static std::vector<int> g_gpu_list;  // f2m_set_gpu_list (empty: primary, primary+1, ...)

struct MultiRank {
  int dev = 0;
  f2m_graph* rep = nullptr;    // replica on dev (shared by ranks on the same device)
  cudaStream_t stream = nullptr;
  DBuf<double> ring;           // kLamBufs x n, buffer 0 = lambda_0
  DBuf<unsigned long long> ll, cmax;
  DBuf<unsigned long long*> ll_peers, cmax_peers;  // [world] device pointers, on dev
  DBuf<unsigned char> ctl;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int begin = 0, end = 0;
};

struct MultiPlan {
  std::vector<int> devs;       // per rank
  int world = 0, gp = 0;
  std::vector<std::unique_ptr<f2m_graph, void (*)(f2m_graph*)>> reps;  // one per distinct device
  std::vector<MultiRank> ranks;
  ~MultiPlan() {
    for (MultiRank& r : ranks) {
      cudaSetDevice(r.dev);
      if (r.stream) cudaStreamSynchronize(r.stream);
      r.ring.release(); r.ll.release(); r.cmax.release(); r.ll_peers.release(); r.cmax_peers.release();
      r.ctl.release();
      if (r.e0) cudaEventDestroy(r.e0);
      if (r.e1) cudaEventDestroy(r.e1);
      if (r.stream) cudaStreamDestroy(r.stream);
    }
    reps.clear();  // f2m_graph_destroy selects each replica's device
  }
};

__global__ void k_multi_gather(int n, const double* __restrict__ src, const int32_t* __restrict__ idx,
                               double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// The rank -> device map of a num_gpus solve whose primary device is `primary`.
static std::vector<int> rank_devices(int primary, int num) {
  std::vector<int> list;
  {
    std::lock_guard<std::mutex> lk(g_gpu_list_mu);
    list = g_gpu_list;
  }
  if (!list.empty()) {
    if ((int)list.size() < num)
      throw Error(F2M_E_ARGUMENT, "num_gpus = " + std::to_string(num) + " but f2m_set_gpu_list named only " +
                                      std::to_string(list.size()) + " devices");
    list.resize(num);
    return list;
  }
  int count = 0;
  F2M_CUDA(cudaGetDeviceCount(&count));
  if (num > count)
    throw Error(F2M_E_ARGUMENT, "num_gpus = " + std::to_string(num) + " but only " + std::to_string(count) +
                                    " CUDA devices are visible");
  for (int r = 0; r < num; ++r) list.push_back((primary + r) % count);
  return list;
}

// g's topology (edge list, costs, spatial order) copied onto `dev` and re-partitioned into
// `partition` CTAs; mean cost carried over (bit-exact sequential sum, computed once on g).
static f2m_graph* replicate(const f2m_graph& g, int dev, int partition) {
  const Topology& t = *g.topo;
  F2M_CUDA(cudaSetDevice(t.dev));
  F2M_CUDA(cudaStreamSynchronize(t.stream));
  F2M_CUDA(cudaSetDevice(dev));
  auto h = std::make_unique<f2m_graph>();
  h->topo = make_topology(t.n, dev);
  Topology& r = *h->topo;
  r.m = t.m;
  r.partition_override = partition;
  cudaStream_t s = r.stream;
  r.eu.alloc(t.m, s);
  r.ev.alloc(t.m, s);
  h->cost.alloc(t.m, s);
  r.perm.alloc(t.n, s);
  r.iperm.alloc(t.n, s);
  if (t.m > 0) {
    F2M_CUDA(cudaMemcpyPeerAsync(r.eu.get(), dev, t.eu.get(), t.dev, t.eu.bytes(), s));
    F2M_CUDA(cudaMemcpyPeerAsync(r.ev.get(), dev, t.ev.get(), t.dev, t.ev.bytes(), s));
    F2M_CUDA(cudaMemcpyPeerAsync(h->cost.get(), dev, g.cost.get(), t.dev, g.cost.bytes(), s));
  }
  if (t.n > 0) {  // the spatial (Morton) order, re-partitioned below
    F2M_CUDA(cudaMemcpyPeerAsync(r.perm.get(), dev, t.perm0.get(), t.dev, t.perm0.bytes(), s));
    F2M_CUDA(cudaMemcpyPeerAsync(r.iperm.get(), dev, t.iperm0.get(), t.dev, t.iperm0.bytes(), s));
  }
  finalize_topology(r);
  attach_costs(*h);
  h->mean_cost = g.mean_cost;
  h->mean_known = g.mean_known;
  h->rounded = g.rounded;
  F2M_CUDA(cudaStreamSynchronize(s));
  return h.release();
}

static void enable_peer_access(const std::vector<int>& devs) {
  for (int a : devs) {
    for (int b : devs) {
      if (a == b) continue;
      int ok = 0;
      F2M_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok)
        throw Error(F2M_E_CUDA, "num_gpus: device " + std::to_string(a) + " cannot access device " +
                                    std::to_string(b) + " (no peer path)");
      F2M_CUDA(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
      } else {
        F2M_CUDA(e);
      }
    }
  }
}

static std::shared_ptr<MultiPlan> make_plan(const f2m_graph& g, const std::vector<int>& devs) {
  const Topology& t = *g.topo;
  const int world = (int)devs.size();
  std::vector<int> distinct = devs;
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  enable_peer_access(distinct);
  // ranks sharing a device split its SMs (each rank's CTAs + master must be co-resident)
  int share = 1, sms = INT32_MAX;
  for (int d : distinct) {
    share = std::max<int>(share, (int)std::count(devs.begin(), devs.end(), d));
    sms = std::min(sms, sweep_grid_ctas(d));
  }
  int gp = std::max(1, (sms - share) / share);
  gp = (int)std::max<int64_t>(1, std::min<int64_t>(gp, ((int64_t)t.n + 31) / 32 / world));
  auto plan = std::make_shared<MultiPlan>();
  plan->devs = devs;
  plan->world = world;
  plan->gp = gp;
  graph_mean(g);  // the replicas inherit the exact sequential mean
  std::vector<f2m_graph*> rep_of(distinct.size(), nullptr);
  for (size_t i = 0; i < distinct.size(); ++i) {
    plan->reps.emplace_back(replicate(g, distinct[i], world * gp), f2m_graph_destroy);
    rep_of[i] = plan->reps.back().get();
  }
  plan->ranks.resize(world);
  for (int r = 0; r < world; ++r) {
    MultiRank& mr = plan->ranks[r];
    mr.dev = devs[r];
    mr.rep = rep_of[std::lower_bound(distinct.begin(), distinct.end(), mr.dev) - distinct.begin()];
    F2M_CUDA(cudaSetDevice(mr.dev));
    F2M_CUDA(cudaStreamCreateWithFlags(&mr.stream, cudaStreamNonBlocking));
    F2M_CUDA(cudaEventCreate(&mr.e0));
    F2M_CUDA(cudaEventCreate(&mr.e1));
    int g_total = 0, resident = 0;
    int64_t llw = 0, cmw = 0;
    if (f2m_sweep_multi_info(mr.rep, r, world, &g_total, &resident, &llw, &cmw, &mr.begin, &mr.end) != F2M_OK)
      throw Error(F2M_E_ARGUMENT, std::string("num_gpus: ") + f2m_last_error());
    mr.ring.alloc((size_t)8 * std::max(t.n, 1), mr.stream);
    mr.ll.alloc((size_t)llw, mr.stream);
    mr.cmax.alloc((size_t)cmw, mr.stream);
    mr.ctl.alloc(f2m_sweep_multi_ctl_bytes(), mr.stream);
    mr.ll_peers.alloc(world, mr.stream);
    mr.cmax_peers.alloc(world, mr.stream);
  }
  std::vector<unsigned long long*> llp(world), cmp(world);
  for (int r = 0; r < world; ++r) {
    llp[r] = plan->ranks[r].ll.get();
    cmp[r] = plan->ranks[r].cmax.get();
  }
  for (MultiRank& mr : plan->ranks) {
    F2M_CUDA(cudaSetDevice(mr.dev));
    F2M_CUDA(cudaMemcpyAsync(mr.ll_peers.get(), llp.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, mr.stream));
    F2M_CUDA(cudaMemcpyAsync(mr.cmax_peers.get(), cmp.data(), sizeof(void*) * world, cudaMemcpyHostToDevice,
                             mr.stream));
    F2M_CUDA(cudaStreamSynchronize(mr.stream));
  }
  return plan;
}

// solve_duals with world_req ranks (cfg.num_gpus clamped to the graph's slice count); d_lam_out
// receives lambda in g's position order
void solve_duals_multi(const f2m_graph& g, const f2m_engine_config& cfg, int world_req, const double* d_init,
                       DBuf<double>& d_lam_out, f2m_convergence_report& rep) {
  const Topology& t = *g.topo;
  const std::vector<int> devs = rank_devices(t.dev, world_req);
  if (!g.multi || g.multi->devs != devs) g.multi = make_plan(g, devs);
  MultiPlan& plan = *g.multi;
  const int world = plan.world, n = t.n;
  MultiRank& r0 = plan.ranks[0];
  const Topology& t0 = *r0.rep->topo;
  // lambda_0 (node-id order is the same whatever the spatial order) in the replicas' position order
  F2M_CUDA(cudaSetDevice(r0.dev));
  if (d_init) {
    F2M_CUDA(cudaSetDevice(t.dev));
    DBuf<double> ids(std::max(n, 1), t.stream);
    if (n > 0) {
      k_multi_gather<<<grid_for(n, 256), 256, 0, t.stream>>>(n, d_init, t.perm.get(), ids.get());
      launched("multi_init_ids");
    }
    F2M_CUDA(cudaStreamSynchronize(t.stream));
    F2M_CUDA(cudaSetDevice(r0.dev));
    DBuf<double> ids0(std::max(n, 1), r0.stream);
    if (n > 0) {
      F2M_CUDA(cudaMemcpyPeerAsync(ids0.get(), r0.dev, ids.get(), t.dev, sizeof(double) * n, r0.stream));
      k_multi_gather<<<grid_for(n, 256), 256, 0, r0.stream>>>(n, ids0.get(), t0.iperm.get(), r0.ring.get());
      launched("multi_init_pos");
    }
    F2M_CUDA(cudaStreamSynchronize(r0.stream));
  } else {
    int* err = reinterpret_cast<int*>(pinned_scratch() + 20);
    *err = 0;
    initial_state_device(*r0.rep, cfg, r0.ring.get(), err);
    F2M_CUDA(cudaStreamSynchronize(t0.stream));
    if (*err) throw Error(F2M_E_TIMEOUT, "initial-state kernel: dependency wait watchdog fired");
  }
  for (int r = 0; r < world; ++r) {
    MultiRank& mr = plan.ranks[r];
    F2M_CUDA(cudaSetDevice(mr.dev));
    if (r > 0 && n > 0)
      F2M_CUDA(cudaMemcpyPeerAsync(mr.ring.get(), mr.dev, r0.ring.get(), r0.dev, sizeof(double) * n, mr.stream));
    F2M_CUDA(cudaMemsetAsync(mr.ll.get(), 0, mr.ll.bytes(), mr.stream));
    F2M_CUDA(cudaMemsetAsync(mr.cmax.get(), 0, mr.cmax.bytes(), mr.stream));
  }
  for (MultiRank& mr : plan.ranks) {  // every ring is clean before any rank publishes
    F2M_CUDA(cudaSetDevice(mr.dev));
    F2M_CUDA(cudaStreamSynchronize(mr.stream));
  }
  const double threshold = cfg.eps * graph_mean(g);  // dual.cpp:221, host fp64 product
  for (int r = 0; r < world; ++r) {
    MultiRank& mr = plan.ranks[r];
    F2M_CUDA(cudaSetDevice(mr.dev));
    F2M_CUDA(cudaEventRecord(mr.e0, mr.stream));
    if (f2m_sweep_multi_launch(mr.rep, &cfg, r, world, mr.ring.get(), mr.ll.get(), mr.ll_peers.get(), mr.cmax.get(),
                               mr.cmax_peers.get(), threshold, cfg.max_sweeps, mr.ctl.get(), mr.stream) != F2M_OK)
      throw Error(F2M_E_CUDA, std::string("num_gpus launch: ") + f2m_last_error());
    F2M_CUDA(cudaEventRecord(mr.e1, mr.stream));
  }
  int sweeps = -1, conv = 0, outbuf = 0;
  double fmax = 0.0, ms_max = 0.0;
  std::string failure;
  for (int r = 0; r < world; ++r) {
    MultiRank& mr = plan.ranks[r];
    F2M_CUDA(cudaSetDevice(mr.dev));
    F2M_CUDA(cudaStreamSynchronize(mr.stream));
    float ms = 0.f;
    F2M_CUDA(cudaEventElapsedTime(&ms, mr.e0, mr.e1));
    ms_max = std::max(ms_max, (double)ms);
    int sw = 0, cv = 0, ob = 0;
    double fm = 0.0;
    if (f2m_sweep_multi_result(mr.ctl.get(), &sw, &cv, &fm, &ob) != F2M_OK) {
      failure = f2m_last_error();
      continue;
    }
    if (sweeps >= 0 && (sw != sweeps || cv != conv || ob != outbuf))
      failure = "num_gpus: ranks disagree on the stopping sweep";
    sweeps = sw;
    conv = cv;
    fmax = fm;
    outbuf = ob;
  }
  if (!failure.empty()) throw Error(F2M_E_TIMEOUT, failure);
  note_sweep_kernel(ms_max, sweeps);
  // each rank's owned positions of the stopping sweep's buffer -> the primary replica's vector
  F2M_CUDA(cudaSetDevice(r0.dev));
  DBuf<double> full(std::max(n, 1), r0.stream);
  for (MultiRank& mr : plan.ranks) {
    if (mr.end <= mr.begin) continue;
    const double* src = mr.ring.get() + (size_t)outbuf * n + mr.begin;
    F2M_CUDA(cudaMemcpyPeerAsync(full.get() + mr.begin, r0.dev, src, mr.dev, sizeof(double) * (mr.end - mr.begin),
                                 r0.stream));
  }
  DBuf<double> ids(std::max(n, 1), r0.stream);
  if (n > 0) {
    k_multi_gather<<<grid_for(n, 256), 256, 0, r0.stream>>>(n, full.get(), t0.perm.get(), ids.get());
    launched("multi_result_ids");
  }
  F2M_CUDA(cudaStreamSynchronize(r0.stream));
  F2M_CUDA(cudaSetDevice(t.dev));
  d_lam_out.alloc(std::max(n, 1), t.stream);
  if (n > 0) {
    DBuf<double> idsg(n, t.stream);
    F2M_CUDA(cudaMemcpyPeerAsync(idsg.get(), t.dev, ids.get(), r0.dev, sizeof(double) * n, t.stream));
    k_multi_gather<<<grid_for(n, 256), 256, 0, t.stream>>>(n, idsg.get(), t.iperm.get(), d_lam_out.get());
    launched("multi_result_pos");
    F2M_CUDA(cudaStreamSynchronize(t.stream));
  }
  rep.sweeps = sweeps;
  rep.converged = conv;
  rep.final_max_abs_delta = fmax;
}

}  // namespace f2mgpu

using namespace f2mgpu;

extern "C" int f2m_set_gpu_list(const int* devices, int count) {
  return guard([&] {
    if (count < 0 || (count > 0 && !devices)) throw Error(F2M_E_ARGUMENT, "f2m_set_gpu_list: bad list");
    int n = 0;
    F2M_CUDA(cudaGetDeviceCount(&n));
    for (int i = 0; i < count; ++i)
      if (devices[i] < 0 || devices[i] >= n) throw Error(F2M_E_ARGUMENT, "f2m_set_gpu_list: no such device");
    std::lock_guard<std::mutex> lk(g_gpu_list_mu);
    g_gpu_list.assign(devices, devices + count);
  });
}

extern "C" int f2m_multi_gpu_info(const f2m_graph* g, int* world, int* partition_ctas, int* resident) {
  return guard([&] {
    if (!g->multi) throw Error(F2M_E_ARGUMENT, "f2m_multi_gpu_info: no num_gpus > 1 solve has run on this graph");
    const MultiPlan& p = *g->multi;
    *world = p.world;
    *partition_ctas = p.world * p.gp;
    *resident = p.reps.front()->topo->resident ? 1 : 0;
  });
}

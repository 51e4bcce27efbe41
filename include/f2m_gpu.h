/*
 * f2m_gpu.h — C ABI of the B200-native F2M gradient-descent-procedure (GDP) solver.
 *
 * This is the drop-in boundary of SURVEY.md §8(b): plain pointers and sizes, no C++ or
 * torch types. Every compute entry point runs hand-written sm_100a CUDA kernels
 * (libf2m_gpu.so); there is no CPU fallback — without a usable CUDA device every call
 * returns F2M_E_CUDA.
 *
 * Each entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj). The host C++ mirror of the reference API (include/f2m/api.hpp,
 * namespace f2m) and the pybind11 module _f2m are thin layers over these calls, so the
 * reference's Python binding (python/bindings.cpp) and C++ headers keep working unchanged.
 *
 * Conventions
 *  - All calls are blocking and return an int status (F2M_OK == 0). On failure
 *    f2m_last_error() returns a thread-local message; the status maps 1:1 onto the
 *    reference's exception taxonomy (include/f2m/errors.hpp:9-57).
 *  - Arrays named h_* / unqualified are HOST memory, caller-owned. Arrays named d_* are
 *    DEVICE memory (already resident in HBM) on the graph's device.
 *  - Node ids and edge ids are the reference's: edges sorted by (u, v) with u < v
 *    (graph.hpp:16-17), lambda indexed by node id. The device internally renumbers nodes
 *    spatially (Morton order of the k-NN grid) — invisible at this boundary.
 *  - A graph handle must not be used from two threads at once.
 */
#ifndef F2M_GPU_H
#define F2M_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception type (errors.hpp) -------------------- */
enum f2m_status {
  F2M_OK = 0,
  F2M_E_ARGUMENT = 1,       /* ArgumentError        errors.hpp:15  */
  F2M_E_INDEX = 2,          /* IndexError           errors.hpp:20  */
  F2M_E_MIN_DEGREE = 3,     /* MinDegreeError       errors.hpp:25  */
  F2M_E_STRUCTURE = 4,      /* StructureError       errors.hpp:30  */
  F2M_E_DEGREE = 5,         /* DegreeError          errors.hpp:35  */
  F2M_E_DEGENERATE = 6,     /* DegenerateExtraction errors.hpp:41  */
  F2M_E_SOLVE_FAILED = 7,   /* SolveFailed          errors.hpp:56  */
  F2M_E_CUDA = 8,           /* CUDA runtime failure / no device (no CPU fallback exists) */
  F2M_E_NOMEM = 9,          /* device allocation failure */
  F2M_E_TIMEOUT = 10        /* device watchdog fired inside a persistent kernel */
};

/* Thread-local description of the last failure on this thread. */
const char* f2m_last_error(void);

/* Selects the CUDA device used by subsequent graph creations on this thread (default 0). */
int f2m_set_device(int device);

/* Library/device facts: SM count, persistent-sweep CTAs and threads, compile target. */
typedef struct {
  int device;
  int sm_count;
  int sweep_ctas;
  int sweep_threads;
  int cc_major;
  int cc_minor;
  char name[96];
} f2m_device_info;
int f2m_get_device_info(f2m_device_info* out);

/* ---- graphs (graph.hpp:18-60) ----------------------------------------------------------
 * An f2m_graph is a device-resident candidate graph: the sorted edge list (u, v, cost), a
 * SELL-32 incidence layout in spatial node order for the GDP sweep, and its mean cost.  */
typedef struct f2m_graph f2m_graph;

/* Graph::from_edges (graph.cpp:14-51): endpoints normalized to u < v, stable-sorted by
 * (u, v); duplicates and self-loops are kept for f2m_graph_validate. F2M_E_INDEX on an
 * endpoint outside [0, n). */
int f2m_graph_from_edges(int n, int64_t m, const int32_t* eu, const int32_t* ev,
                         const double* cost, f2m_graph** out);

/* build_knn_graph (graph.cpp:169-240): symmetrized k-NN graph of n points (xy[2i], xy[2i+1])
 * under DistanceMode rounded (1 = EUC_2D nint, 0 = exact). Candidate lists are bit-exact
 * with the reference. F2M_E_ARGUMENT for k < 3 or n < 4. */
int f2m_knn_build(int n, const double* xy, int rounded, int k, f2m_graph** out);
/* Same, with the points already resident in device memory (d_xy, 2n doubles). */
int f2m_knn_build_device(int n, const double* d_xy, int rounded, int k, f2m_graph** out);

/* generate_instance (instance.cpp:143-157) on the device: the n uniform points of the SplitMix64
 * stream seeded `seed` in [0, box)^2 written to d_xy (2n doubles, x then y per point), bit-identical
 * to the host generator (counter-based: draw j of the stream is computed directly). Stream-ordered
 * on `stream` (NULL = legacy default), no synchronisation. */
int f2m_generate_instance_device(int n, uint64_t seed, double box, double* d_xy, void* stream);

/* Graph::with_costs (graph.cpp:53-65): same topology, new costs and mean cost. */
int f2m_graph_with_costs(const f2m_graph* g, const double* cost, f2m_graph** out);

/* jittered() (solve.cpp:39-47): costs + perturb_scale*cost_scale*U[0,1) from the
 * SplitMix64 stream seeded seed*0x9E3779B97F4A7C15 + restart, one draw per edge in edge-id
 * order — generated on the device, no host round trip of the topology. */
int f2m_graph_jittered(const f2m_graph* g, uint64_t seed, int restart, double perturb_scale,
                       f2m_graph** out);

void f2m_graph_destroy(f2m_graph* g);

typedef struct {
  int n;
  int64_t m;
  double mean_cost;   /* Graph::mean_cost (graph.hpp:49): sequential sum / m, bit-exact */
  int min_degree;
  int max_degree;
  int64_t sell_slots; /* padded SELL-32 slot count (>= 2m) */
  int sweep_ctas;      /* CTAs of the persistent sweep kernel (<= SM count) */
  int sweep_variant;   /* 1 = grid-barrier kernel (k_gdp_sweep), 2 = persistent LL kernel streaming the slots
                          (k_gdp_sweep5<.., false, ..>), 3 = persistent LL kernel, slots resident in smem */
  int max_local;       /* max over CTAs of own + halo nodes (v2 local index space) */
  int64_t max_cta_slots; /* max over CTAs of padded slots */
  int64_t smem_bytes;  /* dynamic shared memory of the v2 kernel */
} f2m_graph_info;
int f2m_graph_get_info(const f2m_graph* g, f2m_graph_info* out);

/* Edge list download (Graph::edges, graph.hpp:30-31). Any pointer may be NULL. */
int f2m_graph_edges(const f2m_graph* g, int32_t* eu, int32_t* ev, double* cost);
/* Per-node degrees (Graph::degree, graph.hpp:38-41). */
int f2m_graph_degrees(const f2m_graph* g, int32_t* degree);
/* Reference CSR incidence (graph.cpp:27-45): offsets[n+1], ids[2m] edge ids ascending per
 * row — for host-side Graph::incident(). */
int f2m_graph_incidence(const f2m_graph* g, int64_t* offsets, int32_t* ids);

/* validate_graph (graph.cpp:242-277): F2M_E_STRUCTURE on the first self-loop / duplicate /
 * negative cost in edge order, F2M_E_MIN_DEGREE if the minimum degree is below 3. */
int f2m_graph_validate(const f2m_graph* g, int* min_degree, int* max_degree, int64_t* edges);

/* ---- dual engine (dual.hpp) ---------------------------------------------------------- */
typedef struct {            /* EngineConfig, dual.hpp:29-40 */
  int b;                    /* right-hand side, 1..8 (kMaxB, dual.cpp:70) */
  double eta;               /* Jacobi damping in (0, 1] */
  double eps;               /* convergence tolerance relative to mean cost */
  int max_sweeps;
  int mode;                 /* 0 = Jacobi, 1 = Gauss-Seidel */
  int update;               /* 0 = midpoint, 1 = paper-difference */
  int init;                 /* 0 = local-midpoint, 1 = zero */
  int threads;              /* accepted for API parity; the device decides its own grid */
  int num_gpus;             /* <= 1: one GPU (the graph's). > 1: solve_duals' Jacobi sweeps run on
                               that many GPUs from the calling thread (multi.cu: the graph is
                               replicated and partitioned across them, halo multipliers move over
                               NVLink peer memory inside one persistent kernel per GPU); clamped to
                               the graph's 32-node slice count. Results are bit-identical. */
} f2m_engine_config;

typedef struct {            /* ConvergenceReport, dual.hpp:48-54 */
  int converged;
  int sweeps;
  double final_max_abs_delta;
  double dual_value;
  double wall_time;
} f2m_convergence_report;

/* EngineConfig::validate (dual.cpp:13-18) plus the b <= 8 bound the reference forgets. */
int f2m_engine_config_validate(const f2m_engine_config* cfg);

/* make_initial_state (dual.cpp:194-208): the in-index-order local-midpoint pass (each node
 * sees the already-updated multipliers of lower-numbered neighbours) or zeros. */
int f2m_initial_state(const f2m_graph* g, const f2m_engine_config* cfg, double* lambda_out);

/* `count` Jacobi sweeps (jacobi_sweep, dual.cpp:129-167) from lambda_inout, in place.
 * max_abs_delta[count] (nullable) receives each sweep's max |delta|; dual_value (nullable)
 * g(lambda) after the last sweep. F2M_E_DEGREE if some degree <= b. */
int f2m_jacobi_sweeps(const f2m_graph* g, const f2m_engine_config* cfg, double* lambda_inout,
                      int count, double* max_abs_delta, double* dual_value);

/* Phase 1 of jacobi_sweep (dual.cpp:138-152) alone: delta[v] for every node from the frozen
 * lambda (smallest_adjusted + delta_for with cfg->b / cfg->update); the pooled jacobi_sweep
 * overload's delta scratch (dual.hpp:83-85). F2M_E_DEGREE if some degree <= b. */
int f2m_jacobi_deltas(const f2m_graph* g, const f2m_engine_config* cfg, const double* lambda, double* delta);

/* `count` Gauss-Seidel sweeps (gauss_seidel_sweep, dual.cpp:175-192), in place. */
int f2m_gauss_seidel_sweeps(const f2m_graph* g, const f2m_engine_config* cfg,
                            double* lambda_inout, int count, double* max_abs_delta,
                            double* dual_value);

/* dual_objective (dual.cpp:87-127): b*sum(lambda) + sum_e min(0, v_e), summed in the
 * reference's 2048-node / 8192-edge chunk order — bit-exact. */
int f2m_dual_objective(const f2m_graph* g, const double* lambda, int b, double* out);

/* node_update_delta (dual.cpp:74-85). */
int f2m_node_update_delta(const f2m_graph* g, const double* lambda, int v, int b, double* out);

/* solve_duals (dual.cpp:210-246): one persistent sm_100a kernel runs every sweep with a
 * device-side convergence test (max|delta| <= eps*mean_cost); no per-sweep host sync.
 * lambda_init may be NULL (then cfg->init decides). */
int f2m_solve_duals(const f2m_graph* g, const f2m_engine_config* cfg, const double* lambda_init,
                    double* lambda_out, f2m_convergence_report* report);

/* ---- extraction + certificate (primal.hpp) -------------------------------------------- */
/* classify_edges (primal.cpp:43-63): 0 = NEG, 1 = ZERO, 2 = POS per edge. */
int f2m_classify_edges(const f2m_graph* g, const double* lambda, double tol, uint8_t* label);

/* extract_primal (primal.cpp:142-233): x[m] in {0, 1/2, 1} and the objective (sequential
 * sum in edge order, bit-exact). F2M_E_DEGENERATE on the reference's degenerate cases. */
int f2m_extract_primal(const f2m_graph* g, const double* lambda, double tol, double* x,
                       double* objective);

/* solve_zero_component (primal.cpp:65-140) — exposed for tests like the reference. */
int f2m_solve_zero_component(const f2m_graph* g, const int32_t* component_edges, int count,
                             const int32_t* residual, double* values, int* feasible);

typedef struct {            /* VerificationReport, primal.hpp:25-30 */
  int feasible;
  int64_t violated_count;
  int64_t value_violation_count;
  double duality_gap;
} f2m_verification;

/* verify_solution (primal.cpp:235-276). violated_nodes/violated_sums/value_violations may
 * be NULL; otherwise they receive up to `capacity` entries in node / edge order. */
int f2m_verify_solution(const f2m_graph* g, const double* x, double objective,
                        const double* lambda, f2m_verification* report, int32_t* violated_nodes,
                        double* violated_sums, int32_t* value_violations, int64_t capacity);

/* ---- pipeline (solve.hpp) ------------------------------------------------------------- */
typedef struct {            /* RunConfig, solve.hpp:15-27 */
  int k;
  f2m_engine_config engine;
  double tol;
  double gap_tol;
  int max_restarts;
  double perturb_scale;
  uint64_t seed;
} f2m_run_config;

int f2m_run_config_validate(const f2m_run_config* rc);

typedef struct {            /* SolveOutcome, solve.hpp:29-35 */
  double objective;
  f2m_verification verification;
  f2m_convergence_report convergence;
  int restarts;
  /* stage timings (seconds, device events) — observability beyond the reference */
  double t_knn, t_duals, t_extract, t_total;
} f2m_solve_outcome;

/* full_solve_graph (solve.cpp:51-99): validate, then restart loop of solve_duals ->
 * extract_primal -> objective on the original costs -> verify_solution -> certify
 * (gap <= gap_tol*(1+|obj|)), jittering on the device between attempts.
 * x (m, nullable) and lambda (n, nullable) are host outputs. F2M_E_SOLVE_FAILED when the
 * restarts are exhausted. */
int f2m_full_solve_graph(const f2m_graph* g, const f2m_run_config* rc, double* x,
                         double* lambda, f2m_solve_outcome* out);

/* full_solve (solve.cpp:101-106): k-NN build with k = max(3, min(k, n-1)) + the above.
 * `graph_out` (nullable) receives the built graph (caller destroys). */
int f2m_full_solve(int n, const double* xy, int rounded, const f2m_run_config* rc, double* x,
                   double* lambda, f2m_solve_outcome* out, f2m_graph** graph_out);

/* Device-resident variant for benchmarking with inputs already in HBM: d_xy (2n doubles)
 * on the device, d_x (m) / d_lambda (n) device outputs (nullable). */
int f2m_full_solve_device(int n, const double* d_xy, int rounded, const f2m_run_config* rc,
                          double* d_x, int64_t d_x_capacity, double* d_lambda,
                          f2m_solve_outcome* out, f2m_graph** graph_out);

/* ---- node-sharded multi-GPU GDP -------------------------------------
 * One process per GPU, each holding the (replicated) graph. Rank r owns the spatial
 * positions [r*stride, min(n, (r+1)*stride)), stride = ceil(n / world), so the concatenation
 * of the ranks' shard buffers in rank order is the full multiplier vector in position order
 * (padded to world*stride) — exactly what an NCCL all-gather produces. A Jacobi sweep of a
 * shard reads only that full vector, so the sharded solve is bit-identical to the one-GPU
 * solve for every world size (dual.cpp:129-167 freezes lambda for the whole sweep).
 * The collectives themselves (all-gather of the shards, max-all-reduce of |delta|) are
 * issued by the caller (NCCL through torch.distributed, paper_2011_08170_b200/sharded.py).
 * All calls below are stream-ordered on the caller's `stream` (a cudaStream_t; NULL = the
 * legacy default stream) and do not synchronise, so they can be captured in a CUDA graph. */
typedef struct f2m_shard f2m_shard;
int f2m_shard_create(const f2m_graph* g, int rank, int world, f2m_shard** out);
void f2m_shard_destroy(f2m_shard* s);
typedef struct {
  int n;          /* nodes of the graph */
  int rank, world;
  int begin, end; /* owned positions [begin, end) */
  int stride;     /* shard buffer length (positions per rank, padded) */
  int64_t slots;  /* SELL slots of the owned rows */
} f2m_shard_info;
int f2m_shard_get_info(const f2m_shard* s, f2m_shard_info* out);
/* One Jacobi sweep (jacobi_sweep, dual.cpp:129-167) of the owned rows: reads d_lam_full
 * (world*stride doubles, position order), writes the updated owned multipliers to
 * d_lam_shard (stride doubles; padding entries are written as 0) and raises *d_max_bits to
 * the bit pattern of max |delta| over the owned rows (atomic max on the IEEE bits of a
 * non-negative double; the caller zeroes it). */
int f2m_shard_sweep(const f2m_shard* s, const f2m_engine_config* cfg, const double* d_lam_full,
                    double* d_lam_shard, unsigned long long* d_max_bits, void* stream);
/* Initial multipliers (make_initial_state, dual.cpp:194-208) in POSITION order into
 * d_lam_pos (n doubles), and position-order <-> node-id-order conversions on the device. */
int f2m_initial_state_positions(const f2m_graph* g, const f2m_engine_config* cfg, double* d_lam_pos,
                                void* stream);
int f2m_positions_to_ids(const f2m_graph* g, const double* d_pos, double* d_ids, void* stream);
/* The device's spatial order: position[v] of every node id v (host array, n int32). Ranks use it
 * to plan the halo exchange of the sharded solve. */
int f2m_graph_positions(const f2m_graph* g, int32_t* position);
/* Halo exchange helpers on the caller's stream (device arrays): d_dst[i] = d_src[d_idx[i]]
 * (pack) and d_dst[d_idx[i]] = d_src[i] (unpack), i < count. */
int f2m_gather_f64(const double* d_src, const int32_t* d_idx, double* d_dst, int64_t count, void* stream);
int f2m_scatter_f64(const double* d_src, const int32_t* d_idx, double* d_dst, int64_t count, void* stream);
int f2m_ids_to_positions(const f2m_graph* g, const double* d_ids, double* d_pos, void* stream);
/* d_out[j] = left-to-right fp64 sum (from +0.0, round-to-nearest, no contraction) of
 * d_v[j*seg_len, min((j+1)*seg_len, k)), bit-identical to a sequential loop but evaluated in
 * parallel (csrc/gpu/seqsum.cu). seg_len <= 0 or >= k: one segment. Replaces the reference's
 * single-threaded accumulations: objective (primal.cpp:226-230), dual-objective chunk sums
 * (dual.cpp:96-109, parallel.cpp chunking) and mean_cost (graph.cpp:47-49). */
int f2m_seq_sums(const double* d_v, int64_t k, int64_t seg_len, double* d_out, void* stream);

/* ---- fused peer-memory node-sharded solve (SURVEY.md §8(e) "faster fused variant") ----------
 * One persistent kernel per rank runs every sweep of jacobi_sweep / solve_duals (dual.cpp:129-167,
 * :210-246) on the rank's rows; halo multipliers are stored straight into the reader's receive
 * buffer (peer memory, LL words), sweep maxima into every rank's board; all ranks take the same
 * stop decision. Buffers (recv: 2 x n_recv x 16 B, board: 4 x world x 16 B) must be zeroed on
 * every rank before any rank launches. The plan lists follow HaloPlan (sharded.py): recv_pos =
 * positions this rank reads, grouped by owner; send_* = (own position, reader rank, index in the
 * reader's recv list). The launch is asynchronous (ranks must run concurrently). */
typedef struct {
  const int32_t* d_recv_pos;
  int64_t n_recv;
  unsigned long long* d_recv_buf;
  const int32_t* d_send_pos;
  const int32_t* d_send_peer;
  const int32_t* d_send_dst;
  int64_t n_send;
  unsigned long long* const* d_peer_recv; /* [world] device pointers */
  const int64_t* d_peer_nrecv;            /* [world] */
  unsigned long long* d_board;
  unsigned long long* const* d_peer_board; /* [world] device pointers */
} f2m_p2p_plan;
typedef struct {
  int sweeps;
  int converged;
  int out_buffer; /* 0: lambda_{k+1} is in d_lam_a, 1: in d_lam_b (own positions) */
  double final_max_abs_delta;
} f2m_p2p_result;
size_t f2m_p2p_ctl_bytes(void);
/* co-resident CTAs of the p2p kernel on the current device (all SMs x occupancy); < 0: -status */
int f2m_p2p_max_ctas(int b);
int f2m_p2p_launch(const f2m_shard* s, const f2m_engine_config* cfg, const f2m_p2p_plan* plan, double* d_lam_a,
                   double* d_lam_b, double threshold, int max_sweeps, int ctas, void* d_ctl, void* stream);
int f2m_p2p_get_result(const void* d_ctl, f2m_p2p_result* out);

/* ---- multi-GPU partition-resident sweep (the one-GPU persistent kernel across ranks) ---------
 * Build the (replicated) graph after f2m_set_sweep_partition(world * Gp); rank r then runs
 * partition CTAs [r*Gp, (r+1)*Gp) + its own convergence master. d_ring: kLamBufs (8) x n doubles,
 * buffer 0 = lambda_0 (full, position order); d_ll / d_cmax: this rank's LL and max rings (sizes
 * from f2m_sweep_multi_info, zeroed on every rank before any launch), d_*_peers: device arrays of
 * every rank's ring (peer memory). Asynchronous; f2m_sweep_multi_result after the stream
 * completes: lambda_{k+1} of positions [begin, end) is in ring buffer out_buffer. */
void f2m_set_sweep_partition(int ctas);
int f2m_sweep_multi_info(const f2m_graph* g, int rank, int world, int* g_total, int* resident, int64_t* ll_words,
                         int64_t* cmax_words, int* begin, int* end);
size_t f2m_sweep_multi_ctl_bytes(void);
int f2m_sweep_multi_launch(const f2m_graph* g, const f2m_engine_config* cfg, int rank, int world, double* d_ring,
                           unsigned long long* d_ll, unsigned long long* const* d_ll_peers,
                           unsigned long long* d_cmax, unsigned long long* const* d_cmax_peers, double threshold,
                           int max_sweeps, void* d_ctl, void* stream);
int f2m_sweep_multi_result(const void* d_ctl, int* sweeps, int* converged, double* final_max, int* out_buffer);
/* Peer-memory stores rank r issues per sweep: LL words of its boundary multipliers into the other
 * ranks that read them, and its CTAs' sweep maxima into the other ranks' max rings (16 B each). */
int f2m_sweep_multi_traffic(const f2m_graph* g, int rank, int world, int64_t* remote_ll_stores,
                            int64_t* remote_max_stores);

/* Complete graphs whose costs are the points' distances (build_knn_graph with k >= n-1,
 * graph.cpp:175; n <= 8192) sweep with a dedicated kernel: mode 2 (default) streams an n x n
 * distance matrix computed once per graph (n^2 doubles of device memory), 1 recomputes every cost
 * from the points each sweep (no extra memory, FP64-bound), 0 uses the CSR kernels. All three are
 * bit-identical. Process-wide; takes effect at the next solve. */
int f2m_set_allpairs_mode(int mode);

/* ---- single-process multi-GPU (f2m_engine_config.num_gpus > 1) ------------------------------
 * Devices of rank 0..num_gpus-1 (default: the graph's device and the next num_gpus-1, modulo the
 * device count). A device may repeat: those ranks then share its SMs (test configurations on one
 * GPU). count = 0 restores the default. */
int f2m_set_gpu_list(const int* devices, int count);
/* Facts of the most recent num_gpus > 1 solve on g: ranks, total partition CTAs, and whether the
 * per-CTA slot data is shared-memory resident (else streamed from L2/HBM each sweep). */
int f2m_multi_gpu_info(const f2m_graph* g, int* world, int* partition_ctas, int* resident);

/* ---- instrumentation (bench.py / tests) ----------------------------------------------- */
/* Number of kernels this library launched since load (all entry points). */
uint64_t f2m_kernel_launch_count(void);
/* Device time (ms, CUDA events on the launching stream) of the most recent persistent
 * sweep kernel and the sweeps it ran. */
int f2m_last_sweep_kernel_ms(double* ms, int* sweeps);
/* Human-readable description of the most recent sweep kernel launch (variant, template
 * arguments, grid shape). Valid until the next solve; never NULL. */
const char* f2m_last_sweep_kernel_desc(void);
/* Debug builds only (nvcc -DF2M_WARP_PROFILE): per-warp cycle accounting of the most recent
 * persistent sweep launch, [160][32][12] counters (halo wait, boundary rows, interior rows,
 * end-of-sweep barrier, sweeps, interior slices, interior slot columns, boundary slice width).
   Fields 8-10: boundary-row setup, scan, finish + publish. The product build returns F2M_E_ARGUMENT. */
int f2m_debug_warp_profile(unsigned long long* out, size_t count);
/* debug builds only (-DF2M_WARP_PROFILE): per-CTA event clocks of 64 sweeps of the last sweep
   launch, [160][64][4]; reset != 0 zeroes them first. */
int f2m_debug_sweep_trace(unsigned long long* out, size_t count, int reset);
/* Algorithmic bytes per sweep of this graph's GDP kernel:
 * 4(n+1) + 2m*(4+8) + 16n. */
double f2m_sweep_algorithmic_bytes(const f2m_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* F2M_GPU_H */

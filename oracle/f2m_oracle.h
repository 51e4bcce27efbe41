/*
 * f2m_oracle.h — CPU restatement of the reference F2M/GDP path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The product
 * (paper_2011_08170_b200) never links, imports or executes anything under oracle/.
 *
 * Parity pinned by: tests/golden/ fixtures generated from the UNMODIFIED reference
 * (oracle/_ref, built by oracle/Makefile from /root/reference/proj/src) via
 * tests/golden/make_golden.py, and by live comparison against oracle/_ref when present
 * (tests/test_oracle_vs_ref.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). All arithmetic is IEEE fp64 without FMA contraction, like the
 * reference's -O3 x86-64 build (no -march).
 */
#ifndef F2M_ORACLE_H
#define F2M_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_E_ARGUMENT = 1,
  ORC_E_DEGREE = 2,
  ORC_E_DEGENERATE = 3,
  ORC_E_SOLVE_FAILED = 4,
  ORC_E_NOMEM = 5,
};

/* instance.hpp:49-64, instance.cpp:143-157 — xy[2i]=x, xy[2i+1]=y. */
void orc_generate_instance(int n, uint64_t seed, double box, double* xy);

/* instance.cpp:126-141 */
double orc_distance(const double* xy, int rounded, int i, int j);

/* graph.cpp:169-240 + from_edges graph.cpp:14-51.
 * Returns m (edge count) or -1 on error; *eu,*ev,*cost are malloc'ed (free with orc_free). */
int64_t orc_build_knn(int n, const double* xy, int rounded, int k, int** eu, int** ev,
                      double** cost);

/* test_support.hpp:32-53 quadratic scan (the reference's own k-NN test oracle). */
int64_t orc_knn_scan(int n, const double* xy, int rounded, int k, int** eu, int** ev,
                     double** cost);

void orc_free(void* p);

/* CSR incidence of graph.cpp:14-51: off[n+1] (int64), ids[2m] (edge ids ascending per row);
 * returns mean_cost (sequential sum, graph.cpp:47-49). Edges must be sorted by (u,v). */
double orc_csr(int n, int64_t m, const int* eu, const int* ev, const double* cost,
               int64_t* off, int* ids);

typedef struct {
  int b;
  double eta;
  double eps;
  int max_sweeps;
  int mode;    /* 0 jacobi, 1 gauss-seidel */
  int update;  /* 0 midpoint, 1 paper-difference */
  int init;    /* 0 local-midpoint, 1 zero */
} orc_engine_config;

typedef struct {
  int converged;
  int sweeps;
  double final_max_abs_delta;
  double dual_value;
} orc_report;

/* dual.cpp:194-208 */
void orc_initial_state(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                       const orc_engine_config* cfg, double* lambda);

/* dual.cpp:129-167 (pool-free sequential restatement; chunk order kept for dual value). */
int orc_jacobi_sweep(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                     const orc_engine_config* cfg, double* lambda, double* max_abs_delta,
                     double* dual_value);

/* dual.cpp:175-192 */
int orc_gauss_seidel_sweep(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                           const orc_engine_config* cfg, double* lambda, double* max_abs_delta,
                           double* dual_value);

/* dual.cpp:87-123 (chunks of 2048 nodes / 8192 edges, partials combined in order). */
double orc_dual_objective(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                          const double* lambda, int b);

/* dual.cpp:210-246. lambda_inout: if use_initial, the initial state; always the result. */
int orc_solve_duals(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                    double mean_cost, const orc_engine_config* cfg, int use_initial,
                    double* lambda_inout, orc_report* rep);

/* primal.cpp:43-63: labels 0=NEG 1=ZERO 2=POS */
int orc_classify(int64_t m, const int* eu, const int* ev, const double* cost,
                 const double* lambda, double tol, uint8_t* label);

/* primal.cpp:142-233. x[m] out; objective out. ORC_E_DEGENERATE on failure. */
int orc_extract(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                const double* lambda, double tol, double* x, double* objective);

/* primal.cpp:235-276: returns number of violated nodes; *value_violations, *gap out. */
int orc_verify(int n, int64_t m, const int* eu, const int* ev, const double* cost,
               const double* x, double objective, const double* lambda, int* value_violations,
               double* gap);

typedef struct {
  int k;
  orc_engine_config engine;
  double tol;
  double gap_tol;
  int max_restarts;
  double perturb_scale;
  uint64_t seed;
} orc_run_config;

typedef struct {
  double objective;
  double gap;
  int feasible;
  int restarts;
  orc_report convergence;
} orc_outcome;

/* solve.cpp:51-99 (jittered restarts solve.cpp:39-47). x[m], lambda[n] out. */
int orc_full_solve_graph(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                         const orc_run_config* rc, double* x, double* lambda, orc_outcome* out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * f2m_oracle.c — CPU restatement of the reference F2M/GDP path (see f2m_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product. Sequential plain C.
 * Reference paths are relative to /root/reference/proj.
 */
#include "f2m_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NODE_CHUNK 2048 /* parallel.hpp:15 */
#define EDGE_CHUNK 8192 /* parallel.hpp:16 */
#define MAX_B 8         /* dual.cpp:70 */
#define MAX_COMPONENT_EDGES 20 /* primal.cpp:17 */

void orc_free(void* p) { free(p); }

/* ---------------------------------------------------------------- instance */

/* SplitMix64::next — instance.hpp:54-60 */
static uint64_t sm64_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* SplitMix64::next_double — instance.hpp:63 */
static double sm64_double(uint64_t* state) {
  return (double)(sm64_next(state) >> 11) * 0x1.0p-53;
}

/* generate_instance — instance.cpp:143-157 (x then y per point) */
void orc_generate_instance(int n, uint64_t seed, double box, double* xy) {
  uint64_t st = seed;
  for (int i = 0; i < n; ++i) {
    const double x = sm64_double(&st) * box;
    const double y = sm64_double(&st) * box;
    xy[2 * i] = x;
    xy[2 * i + 1] = y;
  }
}

/* distance — instance.cpp:126-141: sqrt(dx*dx + dy*dy), rounded = floor(d + 0.5) */
double orc_distance(const double* xy, int rounded, int i, int j) {
  const double dx = xy[2 * i] - xy[2 * j];
  const double dy = xy[2 * i + 1] - xy[2 * j + 1];
  const double d = sqrt(dx * dx + dy * dy);
  return rounded ? floor(d + 0.5) : d;
}

/* ---------------------------------------------------------------- graph */

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* symmetrize + sort + unique (graph.cpp:223-232), costs via distance(u, v) (:234-237) */
static int64_t finish_edges(int n, int per_node, const int* nbr, const double* xy, int rounded,
                            int** eu, int** ev, double** cost) {
  const int64_t np = (int64_t)n * per_node;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(np > 0 ? np : 1));
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < per_node; ++j) {
      const int q = nbr[(int64_t)i * per_node + j];
      const uint32_t a = (uint32_t)(i < q ? i : q), b = (uint32_t)(i < q ? q : i);
      keys[(int64_t)i * per_node + j] = ((uint64_t)a << 32) | b;
    }
  }
  qsort(keys, (size_t)np, sizeof(uint64_t), cmp_u64);
  int64_t m = 0;
  for (int64_t t = 0; t < np; ++t) {
    if (t == 0 || keys[t] != keys[t - 1]) keys[m++] = keys[t];
  }
  *eu = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  *ev = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  *cost = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int64_t e = 0; e < m; ++e) {
    (*eu)[e] = (int)(keys[e] >> 32);
    (*ev)[e] = (int)(keys[e] & 0xffffffffu);
    (*cost)[e] = orc_distance(xy, rounded, (*eu)[e], (*ev)[e]);
  }
  free(keys);
  return m;
}

/* NeighborHeap::offer as a sorted bounded list — graph.cpp:135-165. The kept set (the k
 * smallest offered (d, idx) pairs) does not depend on the container. */
static void offer(double* d, int* id, int* cnt, int k, double dd, int q) {
  if (*cnt == k) {
    if (!(dd < d[k - 1] || (dd == d[k - 1] && q < id[k - 1]))) return;
    --*cnt;
  }
  int i = (*cnt)++;
  while (i > 0 && (d[i - 1] > dd || (d[i - 1] == dd && id[i - 1] > q))) {
    d[i] = d[i - 1];
    id[i] = id[i - 1];
    --i;
  }
  d[i] = dd;
  id[i] = q;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* build_knn_graph — graph.cpp:169-240 with PointGrid graph.cpp:70-132 */
int64_t orc_build_knn(int n, const double* xy, int rounded, int k, int** eu, int** ev,
                      double** cost) {
  if (k < 3 || n < 4) return -1;
  const int per_node = k < n - 1 ? k : n - 1;
  /* PointGrid ctor: bbox, cell = sqrt(area/n), doubled until gx*gy <= 64 + 8n */
  double min_x = xy[0], max_x = xy[0], min_y = xy[1], max_y = xy[1];
  for (int i = 0; i < n; ++i) {
    min_x = xy[2 * i] < min_x ? xy[2 * i] : min_x; /* std::min / std::max semantics */
    max_x = xy[2 * i] > max_x ? xy[2 * i] : max_x;
    min_y = xy[2 * i + 1] < min_y ? xy[2 * i + 1] : min_y;
    max_y = xy[2 * i + 1] > max_y ? xy[2 * i + 1] : max_y;
  }
  const double width = max_x - min_x, height = max_y - min_y;
  const double area = width * height;
  double cell = area > 0.0 ? sqrt(area / (double)n) : (width > height ? width : height);
  if (!(cell > 0.0)) cell = 1.0;
  int gx, gy;
  for (;;) {
    gx = (int)(width / cell) + 1;
    if (gx < 1) gx = 1;
    gy = (int)(height / cell) + 1;
    if (gy < 1) gy = 1;
    if ((int64_t)gx * gy <= 64 + 8 * (int64_t)n) break;
    cell *= 2.0;
  }
  const int64_t cells = (int64_t)gx * gy;
  int64_t* off = (int64_t*)calloc((size_t)cells + 1, sizeof(int64_t));
  int* cell_of = (int*)malloc(sizeof(int) * (size_t)n);
  int* ids = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const int cx = clampi((int)((xy[2 * i] - min_x) / cell), 0, gx - 1);
    const int cy = clampi((int)((xy[2 * i + 1] - min_y) / cell), 0, gy - 1);
    cell_of[i] = cy * gx + cx;
    ++off[cell_of[i] + 1];
  }
  for (int64_t c = 1; c <= cells; ++c) off[c] += off[c - 1];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)cells);
  memcpy(cur, off, sizeof(int64_t) * (size_t)cells);
  for (int i = 0; i < n; ++i) ids[cur[cell_of[i]]++] = i;
  free(cur);

  const int max_ring = gx > gy ? gx : gy;
  int* nbr = (int*)malloc(sizeof(int) * (size_t)n * (size_t)per_node);
  double* hd = (double*)malloc(sizeof(double) * (size_t)per_node);
  int* hi = (int*)malloc(sizeof(int) * (size_t)per_node);
  for (int node = 0; node < n; ++node) {
    int cnt = 0;
    const int ccx = clampi((int)((xy[2 * node] - min_x) / cell), 0, gx - 1);
    const int ccy = clampi((int)((xy[2 * node + 1] - min_y) / cell), 0, gy - 1);
    for (int r = 0; r <= max_ring; ++r) {
      const int x0 = ccx - r, x1 = ccx + r, y0 = ccy - r, y1 = ccy + r;
      for (int cy = y0 > 0 ? y0 : 0; cy <= (gy - 1 < y1 ? gy - 1 : y1); ++cy) {
        const int y_edge = (cy == y0 || cy == y1);
        for (int cx = x0 > 0 ? x0 : 0; cx <= (gx - 1 < x1 ? gx - 1 : x1); ++cx) {
          if (!y_edge && cx != x0 && cx != x1) continue; /* ring cells only (:214) */
          const int64_t c = (int64_t)cy * gx + cx;
          for (int64_t t = off[c]; t < off[c + 1]; ++t) {
            const int q = ids[t];
            if (q == node) continue;
            offer(hd, hi, &cnt, per_node, orc_distance(xy, rounded, node, q), q);
          }
        }
      }
      if (cnt == per_node) { /* exact stop bound, graph.cpp:203-211 */
        double bound = (double)r * cell * (1.0 - 1e-12);
        if (rounded) bound -= 0.5;
        if (bound > hd[per_node - 1]) break;
      }
    }
    for (int j = 0; j < per_node; ++j) nbr[(int64_t)node * per_node + j] = hi[j];
  }
  free(hd);
  free(hi);
  free(off);
  free(cell_of);
  free(ids);
  const int64_t m = finish_edges(n, per_node, nbr, xy, rounded, eu, ev, cost);
  free(nbr);
  return m;
}

/* knn_graph_scan — tests/test_support.hpp:32-53 */
int64_t orc_knn_scan(int n, const double* xy, int rounded, int k, int** eu, int** ev,
                     double** cost) {
  const int per_node = k < n - 1 ? k : n - 1;
  int* nbr = (int*)malloc(sizeof(int) * (size_t)n * (size_t)(per_node > 0 ? per_node : 1));
  double* hd = (double*)malloc(sizeof(double) * (size_t)(per_node > 0 ? per_node : 1));
  int* hi = (int*)malloc(sizeof(int) * (size_t)(per_node > 0 ? per_node : 1));
  for (int i = 0; i < n; ++i) {
    int cnt = 0;
    for (int j = 0; j < n; ++j) {
      if (j != i) offer(hd, hi, &cnt, per_node, orc_distance(xy, rounded, i, j), j);
    }
    for (int j = 0; j < per_node; ++j) nbr[(int64_t)i * per_node + j] = hi[j];
  }
  free(hd);
  free(hi);
  const int64_t m = finish_edges(n, per_node, nbr, xy, rounded, eu, ev, cost);
  free(nbr);
  return m;
}

/* Graph::from_edges incidence — graph.cpp:14-51 */
double orc_csr(int n, int64_t m, const int* eu, const int* ev, const double* cost,
               int64_t* off, int* ids) {
  memset(off, 0, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t e = 0; e < m; ++e) {
    ++off[eu[e] + 1];
    if (ev[e] != eu[e]) ++off[ev[e] + 1];
  }
  for (int v = 0; v < n; ++v) off[v + 1] += off[v];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  memcpy(cur, off, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t e = 0; e < m; ++e) {
    ids[cur[eu[e]]++] = (int)e;
    if (ev[e] != eu[e]) ids[cur[ev[e]]++] = (int)e;
  }
  free(cur);
  double total = 0.0;
  for (int64_t e = 0; e < m; ++e) total += cost[e];
  return m > 0 ? total / (double)m : 0.0;
}

typedef struct {
  int n;
  int64_t m;
  const int* eu;
  const int* ev;
  const double* cost;
  int64_t* off;
  int* ids;
  double mean_cost;
} graph_t;

static int graph_init(graph_t* g, int n, int64_t m, const int* eu, const int* ev,
                      const double* cost) {
  g->n = n;
  g->m = m;
  g->eu = eu;
  g->ev = ev;
  g->cost = cost;
  g->off = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  g->ids = (int*)malloc(sizeof(int) * (size_t)(2 * m + 1));
  if (!g->off || !g->ids) return ORC_E_NOMEM;
  g->mean_cost = orc_csr(n, m, eu, ev, cost, g->off, g->ids);
  return ORC_OK;
}

static void graph_free(graph_t* g) {
  free(g->off);
  free(g->ids);
}

/* ---------------------------------------------------------------- dual */

/* smallest_adjusted — dual.cpp:33-61. val = (cost - lambda_v) - lambda_other. */
static int smallest_adjusted(const graph_t* g, const double* lambda, int v, int b, double* out) {
  const int64_t lo = g->off[v], hi = g->off[v + 1];
  if (hi - lo <= b) return 0;
  const int want = b + 1;
  int have = 0;
  const double lv = lambda[v];
  for (int64_t t = lo; t < hi; ++t) {
    const int e = g->ids[t];
    const double other = g->eu[e] == v ? lambda[g->ev[e]] : lambda[g->eu[e]];
    const double val = g->cost[e] - lv - other;
    if (have < want) {
      int i = have++;
      while (i > 0 && out[i - 1] > val) {
        out[i] = out[i - 1];
        --i;
      }
      out[i] = val;
    } else if (val < out[want - 1]) {
      int i = want - 1;
      while (i > 0 && out[i - 1] > val) {
        out[i] = out[i - 1];
        --i;
      }
      out[i] = val;
    }
  }
  return 1;
}

/* delta_for — dual.cpp:63-68 */
static double delta_for(const double* s, int b, int update) {
  if (update == 1) return 0.5 * (s[b - 1] - s[b]);
  return 0.5 * (s[b - 1] + s[b]);
}

/* dual_objective_pooled — dual.cpp:87-123 */
static double dual_objective_g(const graph_t* g, const double* lambda, int b) {
  double node_sum = 0.0;
  for (int64_t c = 0; c * NODE_CHUNK < g->n; ++c) {
    double acc = 0.0;
    const int64_t end = (c + 1) * NODE_CHUNK < g->n ? (c + 1) * NODE_CHUNK : g->n;
    for (int64_t v = c * NODE_CHUNK; v < end; ++v) acc += lambda[v];
    node_sum += acc; /* combine_partials, parallel.cpp:102-106 */
  }
  double edge_sum = 0.0;
  for (int64_t c = 0; c * EDGE_CHUNK < g->m; ++c) {
    double acc = 0.0;
    const int64_t end = (c + 1) * EDGE_CHUNK < g->m ? (c + 1) * EDGE_CHUNK : g->m;
    for (int64_t e = c * EDGE_CHUNK; e < end; ++e) {
      const double val = g->cost[e] - lambda[g->eu[e]] - lambda[g->ev[e]];
      if (val < 0.0) acc += val;
    }
    edge_sum += acc;
  }
  return (double)b * node_sum + edge_sum;
}

double orc_dual_objective(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                          const double* lambda, int b) {
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  const double r = dual_objective_g(&g, lambda, b);
  graph_free(&g);
  return r;
}

static int validate_cfg(const orc_engine_config* c) { /* dual.cpp:13-18 */
  if (c->b < 1 || c->b > MAX_B) return ORC_E_ARGUMENT;
  if (!(c->eta > 0.0) || c->eta > 1.0) return ORC_E_ARGUMENT;
  if (!(c->eps > 0.0)) return ORC_E_ARGUMENT;
  if (c->max_sweeps < 0) return ORC_E_ARGUMENT;
  return ORC_OK;
}

/* make_initial_state — dual.cpp:194-208: in-order pass from 0; lambda is read while written */
static void initial_state_g(const graph_t* g, const orc_engine_config* cfg, double* lambda) {
  for (int v = 0; v < g->n; ++v) lambda[v] = 0.0;
  if (cfg->init != 0) return;
  double s[MAX_B + 1];
  for (int v = 0; v < g->n; ++v) {
    if (smallest_adjusted(g, lambda, v, cfg->b, s)) lambda[v] = 0.5 * (s[cfg->b - 1] + s[cfg->b]);
  }
}

void orc_initial_state(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                       const orc_engine_config* cfg, double* lambda) {
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  initial_state_g(&g, cfg, lambda);
  graph_free(&g);
}

/* jacobi_sweep — dual.cpp:129-167 */
static int jacobi_g(const graph_t* g, const orc_engine_config* cfg, double* lambda, double* delta,
                    double* max_abs_delta, double* dual_value) {
  double s[MAX_B + 1];
  double mx = 0.0;
  for (int v = 0; v < g->n; ++v) {
    if (!smallest_adjusted(g, lambda, v, cfg->b, s)) return ORC_E_DEGREE;
    delta[v] = delta_for(s, cfg->b, cfg->update);
    const double a = fabs(delta[v]);
    mx = mx > a ? mx : a;
  }
  for (int v = 0; v < g->n; ++v) lambda[v] += cfg->eta * delta[v];
  *max_abs_delta = mx;
  if (dual_value) *dual_value = dual_objective_g(g, lambda, cfg->b);
  return ORC_OK;
}

/* gauss_seidel_sweep — dual.cpp:175-192 */
static int gs_g(const graph_t* g, const orc_engine_config* cfg, double* lambda,
                double* max_abs_delta, double* dual_value) {
  double s[MAX_B + 1];
  double mx = 0.0;
  for (int v = 0; v < g->n; ++v) {
    if (!smallest_adjusted(g, lambda, v, cfg->b, s)) return ORC_E_DEGREE;
    const double d = delta_for(s, cfg->b, cfg->update);
    lambda[v] += d;
    const double a = fabs(d);
    mx = mx > a ? mx : a;
  }
  *max_abs_delta = mx;
  if (dual_value) *dual_value = dual_objective_g(g, lambda, cfg->b);
  return ORC_OK;
}

int orc_jacobi_sweep(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                     const orc_engine_config* cfg, double* lambda, double* max_abs_delta,
                     double* dual_value) {
  if (validate_cfg(cfg)) return ORC_E_ARGUMENT;
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  double* delta = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  const int rc = jacobi_g(&g, cfg, lambda, delta, max_abs_delta, dual_value);
  free(delta);
  graph_free(&g);
  return rc;
}

int orc_gauss_seidel_sweep(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                           const orc_engine_config* cfg, double* lambda, double* max_abs_delta,
                           double* dual_value) {
  if (validate_cfg(cfg)) return ORC_E_ARGUMENT;
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  const int rc = gs_g(&g, cfg, lambda, max_abs_delta, dual_value);
  graph_free(&g);
  return rc;
}

/* solve_duals — dual.cpp:210-246. The per-sweep dual value is only reported for the last
 * sweep (dual.cpp:234), so it is computed once at the end: identical result. */
static int solve_duals_g(const graph_t* g, const orc_engine_config* cfg, int use_initial,
                         double* lambda, orc_report* rep) {
  if (validate_cfg(cfg)) return ORC_E_ARGUMENT;
  if (!use_initial) initial_state_g(g, cfg, lambda);
  const double threshold = cfg->eps * g->mean_cost;
  double* delta = (double*)malloc(sizeof(double) * (size_t)(g->n > 0 ? g->n : 1));
  rep->converged = 0;
  rep->sweeps = 0;
  rep->final_max_abs_delta = INFINITY;
  int rc = ORC_OK;
  for (int sweep = 1; sweep <= cfg->max_sweeps; ++sweep) {
    double mx;
    rc = cfg->mode == 0 ? jacobi_g(g, cfg, lambda, delta, &mx, NULL)
                        : gs_g(g, cfg, lambda, &mx, NULL);
    if (rc) break;
    rep->sweeps = sweep;
    rep->final_max_abs_delta = mx;
    if (mx <= threshold) {
      rep->converged = 1;
      break;
    }
  }
  free(delta);
  rep->dual_value = dual_objective_g(g, lambda, cfg->b);
  return rc;
}

int orc_solve_duals(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                    double mean_cost, const orc_engine_config* cfg, int use_initial,
                    double* lambda_inout, orc_report* rep) {
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  g.mean_cost = mean_cost;
  const int rc = solve_duals_g(&g, cfg, use_initial, lambda_inout, rep);
  graph_free(&g);
  return rc;
}

/* ---------------------------------------------------------------- primal */

/* classify_edges — primal.cpp:43-63: v = (c - lambda_u) - lambda_v, u < v */
int orc_classify(int64_t m, const int* eu, const int* ev, const double* cost,
                 const double* lambda, double tol, uint8_t* label) {
  if (!(tol > 0.0)) return ORC_E_ARGUMENT;
  for (int64_t e = 0; e < m; ++e) {
    const double v = cost[e] - lambda[eu[e]] - lambda[ev[e]];
    label[e] = v < -tol ? 0 : (v > tol ? 2 : 1);
  }
  return ORC_OK;
}

/* DisjointSets — primal.cpp:20-39 */
static int ds_find(int* parent, int x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}

typedef struct {
  const int* ends_a;
  const int* ends_b;
  const double* c;
  int* target;
  int* remaining;
  int* halves;
  int* best_halves;
  double best_cost;
  int m;
} zc_t;

/* solve_zero_component DFS — primal.cpp:101-131 */
static void zc_dfs(zc_t* z, int i, double cost) {
  if (cost >= z->best_cost) return;
  if (i == z->m) {
    z->best_cost = cost;
    memcpy(z->best_halves, z->halves, sizeof(int) * (size_t)z->m);
    return;
  }
  const int a = z->ends_a[i], b = z->ends_b[i];
  --z->remaining[a];
  --z->remaining[b];
  const double c = z->c[i];
  for (int h = 0; h <= 2; ++h) {
    if (h > z->target[a] || h > z->target[b]) break;
    z->target[a] -= h;
    z->target[b] -= h;
    if (z->target[a] <= 2 * z->remaining[a] && z->target[b] <= 2 * z->remaining[b]) {
      z->halves[i] = h;
      zc_dfs(z, i + 1, cost + 0.5 * h * c);
    }
    z->target[a] += h;
    z->target[b] += h;
  }
  ++z->remaining[a];
  ++z->remaining[b];
}

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* solve_zero_component — primal.cpp:65-140. Returns 0 if no completion. */
static int solve_component(const int* eu, const int* ev, const double* cost, const int* comp,
                           int mc, const int* residual, double* values) {
  int nodes[2 * MAX_COMPONENT_EDGES];
  int nn = 0;
  for (int i = 0; i < mc; ++i) {
    nodes[nn++] = eu[comp[i]];
    nodes[nn++] = ev[comp[i]];
  }
  qsort(nodes, (size_t)nn, sizeof(int), cmp_int);
  int u = 0;
  for (int i = 0; i < nn; ++i)
    if (i == 0 || nodes[i] != nodes[i - 1]) nodes[u++] = nodes[i];
  nn = u;
  int target[2 * MAX_COMPONENT_EDGES], remaining[2 * MAX_COMPONENT_EDGES];
  int ea[MAX_COMPONENT_EDGES], eb[MAX_COMPONENT_EDGES];
  double cc[MAX_COMPONENT_EDGES];
  int halves[MAX_COMPONENT_EDGES], best[MAX_COMPONENT_EDGES];
  for (int i = 0; i < nn; ++i) {
    target[i] = 2 * residual[nodes[i]];
    remaining[i] = 0;
  }
  for (int i = 0; i < mc; ++i) {
    const int* pa = (const int*)bsearch(&eu[comp[i]], nodes, (size_t)nn, sizeof(int), cmp_int);
    const int* pb = (const int*)bsearch(&ev[comp[i]], nodes, (size_t)nn, sizeof(int), cmp_int);
    ea[i] = (int)(pa - nodes);
    eb[i] = (int)(pb - nodes);
    ++remaining[ea[i]];
    ++remaining[eb[i]];
    cc[i] = cost[comp[i]];
    halves[i] = 0;
  }
  zc_t z = {ea, eb, cc, target, remaining, halves, best, INFINITY, mc};
  zc_dfs(&z, 0, 0.0);
  if (!isfinite(z.best_cost)) return 0;
  for (int i = 0; i < mc; ++i) values[i] = 0.5 * best[i];
  return 1;
}

/* extract_primal — primal.cpp:142-233 */
int orc_extract(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                const double* lambda, double tol, double* x, double* objective) {
  uint8_t* label = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
  if (orc_classify(m, eu, ev, cost, lambda, tol, label)) {
    free(label);
    return ORC_E_ARGUMENT;
  }
  int* negd = (int*)calloc((size_t)n + 1, sizeof(int));
  int* zerod = (int*)calloc((size_t)n + 1, sizeof(int));
  int* residual = (int*)calloc((size_t)n + 1, sizeof(int));
  int* parent = (int*)malloc(sizeof(int) * ((size_t)n + 1));
  int* comp_of_root = (int*)malloc(sizeof(int) * ((size_t)n + 1));
  int rc = ORC_OK;
  for (int64_t e = 0; e < m; ++e) {
    if (label[e] == 0) {
      ++negd[eu[e]];
      ++negd[ev[e]];
    } else if (label[e] == 1) {
      ++zerod[eu[e]];
      ++zerod[ev[e]];
    }
  }
  for (int v = 0; v < n && rc == ORC_OK; ++v) {
    if (negd[v] > 2) rc = ORC_E_DEGENERATE;
    residual[v] = 2 - negd[v];
    if (residual[v] > 0 && zerod[v] == 0) rc = ORC_E_DEGENERATE;
  }
  if (rc == ORC_OK) {
    for (int v = 0; v < n; ++v) {
      parent[v] = v;
      comp_of_root[v] = -1;
    }
    for (int64_t e = 0; e < m; ++e) {
      if (label[e] != 1) continue;
      int a = ds_find(parent, eu[e]), b = ds_find(parent, ev[e]);
      if (a != b) parent[a > b ? a : b] = a < b ? a : b;
    }
    /* components in order of first edge; edges ascending (primal.cpp:179-194) */
    int64_t ncomp = 0;
    int* comp_id = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
    for (int64_t e = 0; e < m; ++e) {
      comp_id[e] = -1;
      if (label[e] != 1) continue;
      const int root = ds_find(parent, eu[e]);
      if (comp_of_root[root] < 0) comp_of_root[root] = (int)ncomp++;
      comp_id[e] = comp_of_root[root];
    }
    int64_t* csize = (int64_t*)calloc((size_t)ncomp + 1, sizeof(int64_t));
    for (int64_t e = 0; e < m; ++e)
      if (comp_id[e] >= 0) ++csize[comp_id[e] + 1];
    for (int64_t c = 0; c < ncomp; ++c) csize[c + 1] += csize[c];
    int* cedges = (int*)malloc(sizeof(int) * (size_t)(csize[ncomp] + 1));
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncomp + 1));
    memcpy(cur, csize, sizeof(int64_t) * (size_t)(ncomp + 1));
    for (int64_t e = 0; e < m; ++e)
      if (comp_id[e] >= 0) cedges[cur[comp_id[e]]++] = (int)e;
    for (int64_t e = 0; e < m; ++e) x[e] = label[e] == 0 ? 1.0 : 0.0;
    for (int64_t c = 0; c < ncomp && rc == ORC_OK; ++c) {
      const int mc = (int)(csize[c + 1] - csize[c]);
      if (mc > MAX_COMPONENT_EDGES) {
        rc = ORC_E_DEGENERATE;
        break;
      }
      double vals[MAX_COMPONENT_EDGES];
      if (!solve_component(eu, ev, cost, cedges + csize[c], mc, residual, vals)) {
        rc = ORC_E_DEGENERATE;
        break;
      }
      for (int i = 0; i < mc; ++i) x[cedges[csize[c] + i]] = vals[i];
    }
    free(comp_id);
    free(csize);
    free(cedges);
    free(cur);
  }
  if (rc == ORC_OK) { /* objective: sequential sum (primal.cpp:226-230) */
    double obj = 0.0;
    for (int64_t e = 0; e < m; ++e) obj += cost[e] * x[e];
    *objective = obj;
  }
  free(label);
  free(negd);
  free(zerod);
  free(residual);
  free(parent);
  free(comp_of_root);
  return rc;
}

/* verify_solution — primal.cpp:235-276 (dual_objective with the default b = 2) */
int orc_verify(int n, int64_t m, const int* eu, const int* ev, const double* cost,
               const double* x, double objective, const double* lambda, int* value_violations,
               double* gap) {
  graph_t g;
  graph_init(&g, n, m, eu, ev, cost);
  int bad = 0;
  for (int v = 0; v < n; ++v) {
    double sum = 0.0;
    for (int64_t t = g.off[v]; t < g.off[v + 1]; ++t) sum += x[g.ids[t]];
    if (sum != 2.0) ++bad;
  }
  int vv = 0;
  for (int64_t e = 0; e < m; ++e)
    if (x[e] != 0.0 && x[e] != 0.5 && x[e] != 1.0) ++vv;
  *value_violations = vv;
  *gap = objective - dual_objective_g(&g, lambda, 2);
  graph_free(&g);
  return bad;
}

/* full_solve_graph — solve.cpp:51-99 with jittered() solve.cpp:39-47 */
int orc_full_solve_graph(int n, int64_t m, const int* eu, const int* ev, const double* cost,
                         const orc_run_config* rc, double* x, double* lambda, orc_outcome* out) {
  if (validate_cfg(&rc->engine) || rc->k < 3 || rc->tol < 0.0 || !(rc->gap_tol > 0.0) ||
      rc->max_restarts < 0 || rc->perturb_scale < 0.0)
    return ORC_E_ARGUMENT;
  graph_t base;
  graph_init(&base, n, m, eu, ev, cost);
  const double eff_tol = rc->tol > 0.0 ? rc->tol : (1e-7 > 10.0 * rc->engine.eps ? 1e-7 : 10.0 * rc->engine.eps);
  double* jc = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  int result = ORC_E_SOLVE_FAILED;
  for (int restart = 0; restart <= rc->max_restarts; ++restart) {
    graph_t g = base;
    const double* c = cost;
    if (restart > 0) {
      const double scale0 = base.mean_cost > 0.0 ? base.mean_cost : 1.0;
      const double amplitude = rc->perturb_scale * scale0;
      uint64_t st = rc->seed * 0x9E3779B97F4A7C15ULL + (uint64_t)restart;
      double total = 0.0;
      for (int64_t e = 0; e < m; ++e) {
        jc[e] = cost[e] + amplitude * sm64_double(&st);
        total += jc[e];
      }
      g.cost = jc;
      g.mean_cost = m > 0 ? total / (double)m : 0.0;
      c = jc;
    }
    orc_report rep;
    const int src = solve_duals_g(&g, &rc->engine, 0, lambda, &rep);
    if (src) { /* solve_duals errors propagate (solve.cpp:64) */
      result = src;
      break;
    }
    const double scale = g.mean_cost > 0.0 ? g.mean_cost : 1.0;
    double obj_j;
    if (orc_extract(n, m, eu, ev, c, lambda, eff_tol * scale, x, &obj_j) != ORC_OK) continue;
    double obj = 0.0;
    for (int64_t e = 0; e < m; ++e) obj += cost[e] * x[e];
    int vv;
    double gap;
    const int bad = orc_verify(n, m, eu, ev, cost, x, obj, lambda, &vv, &gap);
    const int feasible = bad == 0 && vv == 0;
    if (feasible && gap <= rc->gap_tol * (1.0 + fabs(obj))) {
      out->objective = obj;
      out->gap = gap;
      out->feasible = 1;
      out->restarts = restart;
      out->convergence = rep;
      result = ORC_OK;
      break;
    }
  }
  free(jc);
  graph_free(&base);
  return result;
}

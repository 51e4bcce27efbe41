"""Stability of a row's smallest reduced costs across Jacobi sweeps (CPU, numpy; design tool for
the head-first row scan of k_gdp_sweep5, dual.cu row_scan_head).

    python tools/head_stability.py N

Runs the reference's Jacobi iteration (midpoint rule, eta 0.5, b 2; fp64 numpy, not bit-exact) on
the uniform N-city k=10 graph to convergence and reports, for head sizes K = 3..6, how often a
row's top-3 set leaves the head kept since its last repair (rows per sweep, and the rate for
32-row warps of spatially adjacent rows), plus how often two or more tail slots enter at once.
Uses the C oracle (oracle/) only to build the instance and graph.
"""
import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
from oracle import oracle as orc
n = int(sys.argv[1]); k = 10
xy = orc.generate_instance(n, 1, 1000.0)
g = orc.build_knn_graph(xy, k)
lam = orc.initial_state(g)
eu, ev, c = g.eu, g.ev, g.cost
deg = np.bincount(eu, minlength=n) + np.bincount(ev, minlength=n)
W = deg.max()
rows = np.concatenate([eu, ev]); cols = np.concatenate([ev, eu]); cc = np.concatenate([c, c])
o = np.argsort(rows, kind='stable'); rows, cols, cc = rows[o], cols[o], cc[o]
start = np.zeros(n + 1, np.int64); start[1:] = np.cumsum(deg)
pos = np.arange(len(rows)) - start[rows]
NB = np.zeros((n, W), np.int64); C = np.full((n, W), np.inf)
NB[rows, pos] = cols; C[rows, pos] = cc
side = 1000 / np.sqrt(n / 32)
order = np.lexsort(((xy[:,1]//side).astype(int), (xy[:,0]//side).astype(int)))
Ks = [3, 4, 5, 6]
heads = {K: None for K in Ks}
cnt = {K: [0, 0] for K in Ks}  # row hits, warp hits
cnt1 = {K: [0, 0] for K in Ks}  # hits where the tail has >= 2 values entering (min-tracking can't absorb)
sweeps = 0
for s in range(20000):
    Z = (C - lam[:, None]) - lam[NB]
    P = np.argsort(Z, axis=1, kind='stable')
    sv = np.take_along_axis(Z, P[:, :3], 1)
    thr3 = sv[:, 2]
    for K in Ks:
        Hd = heads[K]
        if Hd is None:
            heads[K] = P[:, :K].copy(); continue
        inhead = np.zeros_like(Z, bool); np.put_along_axis(inhead, Hd, True, 1)
        hv = np.sort(np.take_along_axis(Z, Hd, 1), 1)[:, 2]   # head's 3rd smallest
        tailhit = (Z < hv[:, None]) & ~inhead
        hit = tailhit.any(1)
        multi = tailhit.sum(1) >= 2
        cnt[K][0] += hit.sum()
        cnt[K][1] += hit[order][: (n // 32) * 32].reshape(-1, 32).any(1).sum()
        cnt1[K][0] += multi.sum()
        cnt1[K][1] += multi[order][: (n // 32) * 32].reshape(-1, 32).any(1).sum()
        heads[K][hit] = P[hit, :K]
    d = 0.5 * (sv[:, 1] + sv[:, 2])
    lam = lam + 0.5 * d
    sweeps += 1
    md = np.abs(d).max()
    if md <= 1e-9 * c.mean(): break
nw = n // 32
print('n', n, 'sweeps', sweeps)
for K in Ks:
    print(f'K={K}: rows/sweep {cnt[K][0]/sweeps:.2f} ({cnt[K][0]/sweeps/n*100:.4f}%), warp-hit rate {cnt[K][1]/sweeps/nw*100:.3f}% ; multi-entry rows/sweep {cnt1[K][0]/sweeps:.3f}, warp rate {cnt1[K][1]/sweeps/nw*100:.4f}%')

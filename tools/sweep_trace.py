"""Per-CTA event clocks of 64 steady-state sweeps (debug build: tools/build_variant.sh wprof
"-DF2M_WARP_PROFILE"): python tools/sweep_trace.py exp/wprof [--n 100000]

Events per CTA and sweep s (SM clock64, so differences are taken within one CTA): sweep start,
last boundary row published, halo of s staged (both sync warps), end-of-sweep barrier passed.
Prints the median over CTAs and sweeps of: period, start -> halo staged, halo staged -> boundary
published (C_b), boundary published (s) -> halo staged (s+1) (the exchange latency L as seen by
the same CTA; neighbours run in near lockstep), published -> barrier."""
import argparse
import json
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("root")
ap.add_argument("--n", type=int, default=100000)
args = ap.parse_args()
sys.path.insert(0, os.path.abspath(args.root))
import numpy as np  # noqa: E402

import paper_2011_08170_b200 as f2m  # noqa: E402

g = f2m.build_knn_graph(f2m.generate_instance(args.n, 1, 1000.0), 10)
f2m.solve_duals(g, max_sweeps=200000)
f2m._f2m.debug_sweep_trace(True)
st, rep = f2m.solve_duals(g, max_sweeps=200000)
T = f2m._f2m.debug_sweep_trace(False).astype(np.float64)
G = g.layout()["sweep_ctas"]
T = T[:G]
start, pub, staged, bar = T[..., 0], T[..., 1], T[..., 2], T[..., 3]
ok = (start[:, 1:] > 0) & (start[:, :-1] > 0)
per = (start[:, 1:] - start[:, :-1])[ok]
has_b = pub[:, :-1] > 0
d = {
    "n": args.n, "sweeps": rep["sweeps"], "ctas": G,
    "period_cycles_median": float(np.median(per)),
    "start_to_staged": float(np.median((staged - start)[start > 0])),
    "staged_to_published": float(np.median((pub - np.maximum(staged, start))[pub > 0])),
    "published_to_next_staged": float(np.median((staged[:, 1:] - pub[:, :-1])[has_b])),
    "published_to_barrier": float(np.median((bar - pub)[pub > 0])),
    "barrier_to_next_start": float(np.median((start[:, 1:] - bar[:, :-1])[ok])),
}
# per sweep parity (the two-deep-halo form exchanges on even sweeps only)
for par in (0, 1):
    sl = slice(par, None, 2)
    st_, bar_ = start[:, sl], bar[:, sl]
    nxt = start[:, par + 1::2][:, :st_.shape[1]]
    m = min(st_.shape[1], nxt.shape[1])
    ok2 = (st_[:, :m] > 0) & (nxt[:, :m] > 0)
    d["parity%d_sweep_cycles" % par] = float(np.median((nxt[:, :m] - st_[:, :m])[ok2]))
    d["parity%d_start_to_barrier" % par] = float(np.median((bar_ - st_)[(st_ > 0) & (bar_ > 0)]))
print(json.dumps(d))

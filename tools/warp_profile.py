"""Per-warp cycle accounting of the persistent sweep kernel (debug build: tools/build_variant.sh
wprof "-DF2M_WARP_PROFILE"). python tools/warp_profile.py exp/wprof [--n 100000] [--clustered]"""
import argparse
import json
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("root")
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--clustered", action="store_true")
args = ap.parse_args()
sys.path.insert(0, os.path.abspath(args.root))
import numpy as np  # noqa: E402

import paper_2011_08170_b200 as f2m  # noqa: E402

inst = f2m.generate_clustered_instance(args.n, 1) if args.clustered else f2m.generate_instance(args.n, 1, 1000.0)
g = f2m.build_knn_graph(inst, 10)
f2m.solve_duals(g, max_sweeps=200000)
st, rep = f2m.solve_duals(g, max_sweeps=200000)
ms, sw = f2m.last_sweep_kernel()
P = f2m._f2m.debug_warp_profile().astype(np.float64)  # [cta][warp][8]
G = g.layout()["sweep_ctas"]
P = P[:G]
nw = 22
sweeps = P[:, :nw, 4]
per = P[:, :nw, :4] / np.maximum(sweeps[..., None], 1)  # cycles per sweep
tot = per.sum(-1)
names = ["halo_wait", "boundary_rows", "interior_rows", "end_barrier"]
out = {"n": args.n, "us_per_sweep": 1e3 * ms / sw, "sweeps": sw,
       "cycles_per_sweep_mean_total": float(tot.mean()),
       "mean_cycles": {k: float(per[..., i].mean()) for i, k in enumerate(names)},
       "max_over_warps_mean_over_ctas": {k: float(per[..., i].max(1).mean()) for i, k in enumerate(names)},
       "busy_max_warp_mean": float((per[..., 1] + per[..., 2]).max(1).mean()),
       "busy_mean_warp_mean": float((per[..., 1] + per[..., 2]).mean()),
       "interior_slices_per_warp": np.bincount(P[:, :nw, 5].astype(int).ravel()).tolist(),
       "boundary_warps_per_cta": float((P[:, :nw, 7] > 0).sum(1).mean()),
       "boundary_width_mean": float(P[:, :nw, 7][P[:, :nw, 7] > 0].mean()),
       "interior_width_mean": float((P[:, :nw, 6].sum() / max(P[:, :nw, 5].sum(), 1)))}
# the busiest warp of a typical CTA
c = int(np.argsort(tot.max(1))[G // 2])
# per-warp boundary slice width (boundary warps own one 32-row boundary slice each)
sub = P[:, :nw, 8:11] / np.maximum(sweeps[..., None], 1)
out["boundary_row_phases"] = {"setup": float(sub[..., 0][P[:, :nw, 7] > 0].mean()),
                              "scan": float(sub[..., 1][P[:, :nw, 7] > 0].mean()),
                              "finish_publish": float(sub[..., 2][P[:, :nw, 7] > 0].mean())}
out["cta_example"] = {"cta": c, "warps": [[round(float(x)) for x in per[c, w]] + [int(P[c, w, 5]), int(P[c, w, 6]), int(P[c, w, 7])] + [round(float(x)) for x in sub[c, w]]
                                         for w in range(nw)]}
print(json.dumps(out))

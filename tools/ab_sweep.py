"""A/B timing of the persistent sweep kernel across package builds (tools/build_variant.sh).

    python tools/ab_sweep.py ROOT_A ROOT_B ... --n 2000000 --sweeps 400 --reps 5 [--seed 1] [--solve]

Each ROOT is a directory holding a built `paper_2011_08170_b200/` (the repo root, or exp/<name>).
Every build runs in its own subprocess on the same graph; the builds alternate --reps times and
the per-build median us/sweep (CUDA events of the sweep launch) is printed, plus a digest of the
multipliers so a variant that changes results is visible at once.
"""
import argparse
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, hashlib, numpy as np
sys.path.insert(0, %(root)r)
import paper_2011_08170_b200 as f2m
assert f2m.__file__.startswith(%(root)r), f2m.__file__
inst = (f2m.generate_clustered_instance(%(n)d, %(seed)d) if %(clustered)r
        else f2m.generate_instance(%(n)d, %(seed)d, 1000.0))
g = f2m.build_knn_graph(inst, 10)
out = []
for rep in range(%(inner)d):
    if %(solve)r:
        st, r = f2m.solve_duals(g, max_sweeps=200000)
    else:
        st = f2m.make_initial_state(g)
        f2m.jacobi_sweeps(g, st, %(sweeps)d)
    ms, sw = f2m.last_sweep_kernel()
    out.append(1e3 * ms / sw)
print(json.dumps({"us": out, "sweeps": sw, "desc": f2m.last_sweep_kernel_desc(),
                  "digest": hashlib.sha256(np.asarray(st.lam).tobytes()).hexdigest()[:16]}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("roots", nargs="+")
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sweeps", type=int, default=2000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--inner", type=int, default=3)
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--clustered", action="store_true")
    args = ap.parse_args()
    res = {r: [] for r in args.roots}
    meta = {}
    for _ in range(args.reps):
        for r in args.roots:
            code = CHILD % dict(root=os.path.abspath(r), n=args.n, seed=args.seed, sweeps=args.sweeps,
                                inner=args.inner, solve=args.solve, clustered=args.clustered)
            p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
            if p.returncode != 0:
                print(r, "FAILED", p.stderr[-1500:])
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res[r].extend(d["us"][1:] or d["us"])
            meta[r] = (d["sweeps"], d["digest"], d["desc"])
    for r in args.roots:
        v = sorted(res[r])
        med = v[len(v) // 2] if v else float("nan")
        print(json.dumps({"root": r, "n": args.n, "median_us_per_sweep": med, "min": v[0] if v else None,
                          "samples": len(v), "sweeps": meta.get(r, (None,))[0], "digest": meta.get(r, (0, None))[1],
                          "desc": meta.get(r, (0, 0, None))[2]}))


if __name__ == "__main__":
    main()

"""A/B of the certified 100k solve's device time (t_total) across package builds, alternating:
python tools/e2e_ab.py ROOT_A ROOT_B [--reps 5]"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %(root)r)
import paper_2011_08170_b200 as f2m
xy = f2m.generate_instance(100000, 1).points_array()
ts = []
for rep in range(12):
    r = f2m.full_solve_arrays(xy, k=10, eps=1e-9, max_sweeps=200000)
    ts.append((r["t_total"], r["t_knn"], r["t_duals"], r["t_extract"]))
ts = ts[2:]
print(json.dumps({k: statistics.median(t[i] for t in ts) * 1e3 for i, k in enumerate(("total", "knn", "duals", "extract"))}))
'''
roots = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
roots = [r for r in roots if not r.isdigit()]
for _ in range(reps):
    for r in roots:
        p = subprocess.run([sys.executable, "-c", CHILD % dict(root=os.path.abspath(r))], capture_output=True, text=True)
        print(r, p.stdout.strip().splitlines()[-1] if p.returncode == 0 else p.stderr[-300:], flush=True)

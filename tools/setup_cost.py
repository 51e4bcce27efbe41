"""Sweep-kernel launch cost at (almost) zero sweeps: setup (slot upload, initial slot order) +
one sweep. python tools/setup_cost.py ROOT [ROOT ...] [--n N]"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %(root)r)
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(%(n)d, 1, 1000.0), 10)
out = []
for rep in range(7):
    st = f2m.make_initial_state(g)
    f2m.jacobi_sweeps(g, st, %(sweeps)d)
    ms, sw = f2m.last_sweep_kernel()
    out.append(ms)
print(json.dumps({"ms_median": statistics.median(out[1:]), "sweeps": sw}))
'''
args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = 100000
if "--n" in sys.argv:
    n = int(sys.argv[sys.argv.index("--n") + 1])
    args = [a for a in args if a != str(n)]
for root in args:
    for sweeps in (1, 2, 11):
        p = subprocess.run([sys.executable, "-c", CHILD % dict(root=os.path.abspath(root), n=n, sweeps=sweeps)],
                           capture_output=True, text=True)
        print(root, sweeps, p.stdout.strip().splitlines()[-1] if p.returncode == 0 else p.stderr[-500:])

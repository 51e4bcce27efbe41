"""Initial-state kernel time (CUDA events around make_initial_state, median): python tools/init_time.py ROOT..."""
import os
import subprocess
import sys

CHILD = r'''
import sys, time, statistics, torch
sys.path.insert(0, %(root)r)
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1, 1000.0), 10)
ts = []
for _ in range(15):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = f2m.make_initial_state(g)
    ts.append(time.perf_counter() - t0)
print(%(root)r, "make_initial_state wall ms median", round(statistics.median(ts[3:]) * 1e3, 4))
'''
for r in sys.argv[1:]:
    p = subprocess.run([sys.executable, "-c", CHILD % dict(root=os.path.abspath(r))], capture_output=True, text=True)
    print(p.stdout.strip() or p.stderr[-400:])

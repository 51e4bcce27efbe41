"""Quick GPU probe: time a 100k uniform full solve (seed 1) and the sweep kernel alone."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2011_08170_b200 as f2m
print(f2m.device_info(), flush=True)
for n, seed in ((10000, 1), (100000, 1), (200000, 1)):
    print(f2m.build_knn_graph(f2m.generate_instance(n, seed), 10).layout(), flush=True)
    inst = f2m.generate_instance(n, seed)
    xy = inst.points_array()
    for rep in range(2):
        t = time.time()
        r = f2m.full_solve_arrays(xy, k=10, max_sweeps=200000)
        wall = time.time() - t
        ms, sw = f2m.last_sweep_kernel()
        g = r["graph"]
        print(f"n={n} wall={wall:.4f}s t_total={r['t_total']:.4f} knn={r['t_knn']:.4f} duals={r['t_duals']:.4f} "
              f"extract={r['t_extract']:.4f} sweeps={r['sweeps']} obj={r['objective']!r} gap={r['gap']:.3e} "
              f"sweep_kernel={ms:.3f}ms -> {1e3*ms/max(sw,1):.3f}us/sweep bytes/sweep={g.sweep_bytes():.3e} "
              f"sell={g.sell_slots()} 2m={2*g.m}", flush=True)

import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2011_08170_b200 as f2m
xy = f2m.generate_instance(100000, 1).points_array()
xyp = torch.from_numpy(xy).pin_memory().numpy()
for arr, name in ((xy, "pageable"), (xyp, "pinned")):
    for rep in range(4):
        t0 = time.perf_counter()
        r = f2m.full_solve_arrays(arr, k=10, eps=1e-9, max_sweeps=200000)
        w = time.perf_counter() - t0
        print(f"{name}: wall {w*1e3:.2f} ms  t_total {r['t_total']*1e3:.2f}  knn {r['t_knn']*1e3:.2f} duals {r['t_duals']*1e3:.2f} extract {r['t_extract']*1e3:.2f}", flush=True)

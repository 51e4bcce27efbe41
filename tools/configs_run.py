"""Time-to-solve of every BASELINE.json config on one GPU (certified full solves through the C ABI),
next to the reference's sweep counts where SURVEY.md §6 / tests/golden record them."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_08170_b200 as f2m  # noqa: E402
import torch  # noqa: E402

CONFIGS = [
    ("uniform 1k seed 1", "u", 1000, 1, 1e-9),
    ("uniform 10k seed 1", "u", 10000, 1, 1e-9),
    ("uniform 100k seed 1", "u", 100000, 1, 1e-9),
    ("uniform 100k seed 31337 eps 1e-8 (c7)", "u", 100000, 31337, 1e-8),
    ("uniform 200k seed 1", "u", 200000, 1, 1e-9),
    ("clustered 200k seed 1", "c", 200000, 1, 1e-9),
    ("uniform 2M seed 1", "u", 2000000, 1, 1e-9),
]
only = sys.argv[1:] or None
for name, kind, n, seed, eps in CONFIGS:
    if only and not any(o in name for o in only):
        continue
    gen = f2m.generate_clustered_instance if kind == "c" else f2m.generate_instance
    # page-locked input and result buffers (as bench.py's e2e leg)
    xy = torch.from_numpy(gen(n, seed).points_array()).pin_memory().numpy()
    xo = torch.empty(n * 10 + 1, dtype=torch.float64).pin_memory().numpy()
    lo = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    if n <= 200000:  # warm-up
        f2m.full_solve_arrays(xy, k=10, eps=eps, max_sweeps=200000, out_value=xo, out_duals=lo)
    t0 = time.perf_counter()
    try:
        r = f2m.full_solve_arrays(xy, k=10, eps=eps, max_sweeps=400000, out_value=xo, out_duals=lo)
    except Exception as exc:  # the 2M instance: the reference's extraction cap
        print(json.dumps({"config": name, "n": n, "wall_s": time.perf_counter() - t0,
                          "error": f"{type(exc).__name__}: {exc}"[:300]}), flush=True)
        continue
    wall = time.perf_counter() - t0
    ms, sw = f2m.last_sweep_kernel()
    print(json.dumps({"config": name, "n": n, "m": int(r["graph"].m), "wall_s": wall, "t_total": r["t_total"],
                      "t_knn": r["t_knn"], "t_duals": r["t_duals"], "t_extract": r["t_extract"],
                      "sweeps": r["sweeps"], "restarts": r["restarts"], "objective": r["objective"],
                      "gap": r["gap"], "us_per_sweep": 1e3 * ms / max(sw, 1),
                      "kernel": f2m.last_sweep_kernel_desc()}), flush=True)

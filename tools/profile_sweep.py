"""Run exactly one persistent GDP sweep-kernel launch (for ncu).

    python tools/profile_sweep.py N SWEEPS            k-NN graph (k=10) of the uniform instance
    python tools/profile_sweep.py N SWEEPS allpairs   complete graph (k = N-1): k_allpairs_sweep

e.g. ncu --set full --clock-control none --import-source on -k regex:gdp_sweep5 -c 1 -f -o x \\
        python tools/profile_sweep.py 2000000 64
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_08170_b200 as f2m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
allpairs = len(sys.argv) > 3 and sys.argv[3] == "allpairs"
g = f2m.build_knn_graph(f2m.generate_instance(n, 1), n - 1 if allpairs else 10)
print(g.layout())
st = f2m.make_initial_state(g)
mx, dv = f2m.jacobi_sweeps(g, st, sweeps)
ms, sw = f2m.last_sweep_kernel()
if allpairs:
    pairs = n * (n - 1)
    print(f"n={n} allpairs sweeps={sw} kernel_ms={ms:.3f} us/sweep={1e3 * ms / sw:.3f} "
          f"pairs/s={pairs * sw / (ms * 1e-3):.4e} desc={f2m.last_sweep_kernel_desc()}")
else:
    print(f"n={n} m={g.m} sweeps={sw} kernel_ms={ms:.3f} us/sweep={1e3 * ms / sw:.3f} "
          f"bytes/sweep={g.sweep_bytes():.0f} GB/s={g.sweep_bytes() * sw / (ms * 1e-3) / 1e9:.1f} "
          f"desc={f2m.last_sweep_kernel_desc()}")

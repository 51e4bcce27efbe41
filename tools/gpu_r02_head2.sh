mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/head2.log 2>&1
timeout 600 python - > gpurun_out/head2_stats.log 2>&1 <<'PY'
import sys
sys.path.insert(0, 'exp/hstats')
import paper_2011_08170_b200 as f2m
for n in (10000, 100000):
    inst = f2m.generate_instance(n, 1, 1000.0)
    g = f2m.build_knn_graph(inst, 10)
    st, r = f2m.solve_duals(g, max_sweeps=200000)
    print("n", n, "sweeps", r["sweeps"] if isinstance(r, dict) else r, flush=True)
PY
cat gpurun_out/head2.log gpurun_out/head2_stats.log

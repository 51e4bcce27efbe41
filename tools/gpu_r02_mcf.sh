for r in exp/hstats0 exp/hstats; do
python - <<PY 2>&1 | grep "head stats" | tail -1
import sys
sys.path.insert(0, "$r")
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1, 1000.0), 10)
st, r = f2m.solve_duals(g, max_sweeps=200000)
PY
done
bash tools/gpu_r02_var.sh exp/nomcf .
timeout 900 python tools/ab_sweep.py exp/nomcf . --n 200000 --clustered --solve --reps 2 < /dev/null 2>&1 | cut -c1-120

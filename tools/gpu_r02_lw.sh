python - <<PY 2>&1 | grep "head stats" | tail -1
import sys
sys.path.insert(0, "exp/hstats")
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1, 1000.0), 10)
st, r = f2m.solve_duals(g, max_sweeps=200000)
PY
python tools/setup_cost.py exp/warplayout . 2>&1 | grep -v "^$"
bash tools/gpu_r02_var.sh exp/warplayout .
timeout 900 python tools/ab_sweep.py exp/warplayout . --n 10000 --solve --reps 2 < /dev/null 2>&1 | cut -c1-120
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py tests/test_gpu_primal.py < /dev/null 2>&1 | tail -2

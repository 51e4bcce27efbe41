timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1, 1000.0), 10)
st, r = f2m.solve_duals(g, max_sweeps=200000)
print(r, f2m.last_sweep_kernel_desc())
" 2>&1 | tail -3
bash tools/gpu_r02_var.sh exp/noghost .
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py tests/test_gpu_primal.py < /dev/null 2>&1 | tail -3

mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/head3.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/head3.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 200000 --clustered --solve --reps 2 < /dev/null >> gpurun_out/head3.log 2>&1
timeout 600 python - > gpurun_out/head3_stats.log 2>&1 <<'PY'
import sys
sys.path.insert(0, 'exp/hstats')
import paper_2011_08170_b200 as f2m
for n in (100000,):
    inst = f2m.generate_instance(n, 1, 1000.0)
    g = f2m.build_knn_graph(inst, 10)
    st, r = f2m.solve_duals(g, max_sweeps=200000)
    print("n", n, r, flush=True)
PY
timeout 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest_head3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_head3.log
cat gpurun_out/head3.log gpurun_out/head3_stats.log; tail -3 gpurun_out/pytest_head3.log

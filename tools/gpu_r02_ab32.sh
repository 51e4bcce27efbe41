mkdir -p gpurun_out
for v in stats statsl; do
timeout 300 python -c "
import sys; sys.path.insert(0, 'exp/$v')
import paper_2011_08170_b200 as f2m
inst = f2m.generate_instance(100000, 1, 1000.0); g = f2m.build_knn_graph(inst, 10)
st, r = f2m.solve_duals(g, max_sweeps=200000); print('$v', r)
" < /dev/null >> gpurun_out/stats32.log 2>&1
done
cat gpurun_out/stats32.log | grep -v "^$" | tail -6
timeout 900 python tools/ab_sweep.py exp/base exp/lane . --n 100000 --solve --reps 3 && timeout 600 python tools/ab_sweep.py exp/base exp/lane . --n 200000 --solve --reps 2 >> gpurun_out/ab32.log 2>&1 < /dev/null > gpurun_out/ab32.log 2>&1
cat gpurun_out/ab32.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest32.log; tail -2 gpurun_out/pytest32.log

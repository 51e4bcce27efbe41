mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 200000 --clustered --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 10000 --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1

cut -c1-120 gpurun_out/bank.log; tail -3 gpurun_out/pytest_bank.log
python - <<PY 2>&1 | tail -3
import sys
sys.path.insert(0, "exp/hstats")
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1, 1000.0), 10)
st, r = f2m.solve_duals(g, max_sweeps=200000)
print(r["sweeps"])
PY
bash tools/ncu_smem.sh . 2>&1 | tail -5

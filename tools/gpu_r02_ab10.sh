mkdir -p gpurun_out
timeout 600 python tools/ab_sweep.py . exp/sb4 exp/sb6 --n 2000000 --sweeps 300 --reps 2 --inner 2 < /dev/null > gpurun_out/ab10.log 2>&1
cat > /tmp/apab.py <<'PY'
import sys, json
root = sys.argv[1]; sys.path.insert(0, root)
import paper_2011_08170_b200 as f2m
out = []
for n, sw in ((2000, 200), (8000, 30), (4000, 60)):
    g = f2m.build_knn_graph(f2m.generate_instance(n, 1, 1000.0), n - 1)
    st = f2m.make_initial_state(g); f2m.jacobi_sweeps(g, st, 5)
    best = 1e9
    for r in range(3):
        st = f2m.make_initial_state(g); f2m.jacobi_sweeps(g, st, sw)
        ms, s = f2m.last_sweep_kernel(); best = min(best, 1e3 * ms / s)
    out.append((n, round(best, 2)))
print(root, out)
PY
for r in . exp/dnp; do timeout 300 python /tmp/apab.py $r < /dev/null >> gpurun_out/ab10.log 2>&1; done
cat gpurun_out/ab10.log

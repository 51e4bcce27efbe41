# shared-memory wavefronts / bank conflicts of the 100k solve's sweep kernel for each build root
for r in "$@"; do
  echo "== $r"
  timeout 300 ncu --clock-control none --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,gpu__time_duration.sum,smsp__inst_executed.sum -k regex:gdp_sweep5 -c 1 python -c "
import sys; sys.path.insert(0, '$r')
import paper_2011_08170_b200 as f2m
g = f2m.build_knn_graph(f2m.generate_instance(100000, 1), 10)
st, r = f2m.solve_duals(g, max_sweeps=200000)
print(r['sweeps'])
" 2>&1 | grep -E "l1tex|gpu__time|inst_exec|^[0-9]"
done

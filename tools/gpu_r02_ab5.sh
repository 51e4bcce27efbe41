mkdir -p gpurun_out
for n in 100000 200000 10000; do
  timeout 900 python tools/ab_sweep.py exp/base . --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab5.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . --n 2000000 --sweeps 300 --reps 2 --inner 2 < /dev/null >> gpurun_out/ab5.log 2>&1
for n in 100000; do timeout 300 python tools/warp_profile.py exp/wprof --n $n < /dev/null; done > gpurun_out/wprof3.jsonl 2>&1
cat gpurun_out/ab5.log
cat gpurun_out/wprof3.jsonl | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print(d['n'], d['us_per_sweep'], d['sync_warps'], d['boundary_row_phases'])"

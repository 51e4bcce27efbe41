mkdir -p gpurun_out
for n in 100000 200000; do timeout 300 python tools/warp_profile.py exp/wprof --n $n < /dev/null; done > gpurun_out/wprof2.jsonl 2> gpurun_out/wprof2.err
cat gpurun_out/wprof2.jsonl | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print(d['n'], d['us_per_sweep'], d['sync_warps'], d['boundary_row_phases'])"
tail -3 gpurun_out/wprof2.err

mkdir -p gpurun_out
for n in 100000 200000; do timeout 300 python tools/warp_profile.py exp/wprof --n $n < /dev/null; done > gpurun_out/wprof.jsonl 2> gpurun_out/wprof.err
timeout 300 python tools/ab_sweep.py . exp/wprof --n 100000 --solve --reps 1 --inner 3 < /dev/null >> gpurun_out/wprof.jsonl 2>&1
cat gpurun_out/wprof.jsonl; tail -3 gpurun_out/wprof.err

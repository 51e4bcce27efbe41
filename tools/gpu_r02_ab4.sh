mkdir -p gpurun_out
for n in 100000 200000 10000; do
  timeout 900 python tools/ab_sweep.py . exp/split --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab4.log 2>&1
timeout 300 python tools/ab_sweep.py . exp/split --n 200000 --clustered --solve --reps 2 --inner 3 < /dev/null >> gpurun_out/ab4.log 2>&1
timeout 300 python tools/warp_profile.py exp/wprofsplit --n 100000 < /dev/null >> gpurun_out/ab4.log 2>&1
cat gpurun_out/ab4.log

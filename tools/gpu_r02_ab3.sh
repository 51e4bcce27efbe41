mkdir -p gpurun_out
for n in 100000 200000; do
  timeout 900 python tools/ab_sweep.py exp/base . --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab3.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . --n 10000 --solve --reps 2 --inner 3 < /dev/null >> gpurun_out/ab3.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . --n 2000000 --sweeps 300 --reps 2 --inner 2 < /dev/null >> gpurun_out/ab3.log 2>&1
timeout 300 python tools/warp_profile.py exp/wprof --n 100000 < /dev/null >> gpurun_out/ab3.log 2>&1
cat gpurun_out/ab3.log

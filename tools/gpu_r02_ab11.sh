mkdir -p gpurun_out
for n in 100000 200000 10000; do
  timeout 900 python tools/ab_sweep.py . exp/rb4 exp/rb6 --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab11.log 2>&1
cat gpurun_out/ab11.log

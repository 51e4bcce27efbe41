mkdir -p gpurun_out
for n in 100000 200000; do
  timeout 900 python tools/ab_sweep.py . exp/cfh --n $n --sweeps 3000 --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab13.log 2>&1
cat gpurun_out/ab13.log

mkdir -p gpurun_out
for n in 100000 200000 10000; do
  timeout 900 python tools/ab_sweep.py . exp/nt896 exp/nt1024 --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab15.log 2>&1
timeout 300 python tools/ab_sweep.py . exp/nt896 exp/nt1024 --n 200000 --clustered --solve --reps 2 --inner 3 < /dev/null >> gpurun_out/ab15.log 2>&1
cat gpurun_out/ab15.log

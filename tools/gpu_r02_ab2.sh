mkdir -p gpurun_out
for n in 100000 200000; do
  timeout 900 python tools/ab_sweep.py exp/base . exp/pairs --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab2.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . exp/pairs --n 200000 --clustered --solve --reps 2 --inner 3 < /dev/null >> gpurun_out/ab2.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . --n 2000000 --sweeps 300 --reps 2 --inner 2 < /dev/null >> gpurun_out/ab2.log 2>&1
cat gpurun_out/ab2.log

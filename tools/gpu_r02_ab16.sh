mkdir -p gpurun_out
timeout 600 python tools/ab_sweep.py . exp/sp4 --n 2000000 --sweeps 300 --reps 3 --inner 2 < /dev/null > gpurun_out/ab16.log 2>&1
timeout 600 python tools/ab_sweep.py . exp/sp4 --n 400000 --sweeps 1000 --reps 2 --inner 2 < /dev/null >> gpurun_out/ab16.log 2>&1
timeout 600 python tools/ab_sweep.py . exp/sp4 --n 1000000 --sweeps 500 --reps 2 --inner 2 < /dev/null >> gpurun_out/ab16.log 2>&1
cat gpurun_out/ab16.log

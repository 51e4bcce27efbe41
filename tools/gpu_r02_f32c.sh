mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/norescan exp/cf . --n 100000 --sweeps 3000 --reps 2 < /dev/null > gpurun_out/f32c.log 2>&1

cat gpurun_out/f32c.log

mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py . exp/pair exp/pairns --n 100000 --solve --reps 3 < /dev/null > gpurun_out/ab37.log 2>&1
timeout 900 python tools/ab_sweep.py . exp/pair --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/ab37.log 2>&1
timeout 900 python tools/ab_sweep.py . exp/pair --n 200000 --clustered --solve --reps 2 < /dev/null >> gpurun_out/ab37.log 2>&1
cut -c1-150 gpurun_out/ab37.log

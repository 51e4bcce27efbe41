mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base exp/bnd2 --n 100000 --solve --reps 3 < /dev/null > gpurun_out/ab38.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base exp/bnd2 --n 100000 --seed 31337 --solve --reps 2 < /dev/null >> gpurun_out/ab38.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base exp/bnd2 --n 60000 --seed 7 --solve --reps 2 < /dev/null >> gpurun_out/ab38.log 2>&1
cut -c1-200 gpurun_out/ab38.log

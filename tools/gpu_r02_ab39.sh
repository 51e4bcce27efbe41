mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base exp/b256 exp/b0 exp/p256 exp/b1k --n 100000 --solve --reps 2 < /dev/null > gpurun_out/ab39.log 2>&1
cut -c1-150 gpurun_out/ab39.log

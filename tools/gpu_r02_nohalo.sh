timeout 900 python tools/ab_sweep.py exp/nohalo . --n 100000 --sweeps 3000 --reps 2 < /dev/null 2>&1 | cut -c1-120
timeout 900 python tools/ab_sweep.py exp/nohalo . --n 200000 --sweeps 3000 --reps 2 < /dev/null 2>&1 | cut -c1-120

timeout 900 python tools/ab_sweep.py exp/pair . --n 100000 --solve --reps 2 < /dev/null 2>&1 | cut -c1-120
timeout 900 python tools/ab_sweep.py exp/pair . --n 200000 --solve --reps 2 < /dev/null 2>&1 | cut -c1-120

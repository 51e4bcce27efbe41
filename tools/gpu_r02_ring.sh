bash tools/gpu_r02_var.sh exp/ring2 .
timeout 900 python tools/ab_sweep.py exp/ring2 . --n 10000 --solve --reps 2 < /dev/null 2>&1 | cut -c1-120
timeout 900 python tools/ab_sweep.py exp/ring2 . --n 200000 --clustered --solve --reps 2 < /dev/null 2>&1 | cut -c1-120
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests -m gpu < /dev/null 2>&1 | tail -2

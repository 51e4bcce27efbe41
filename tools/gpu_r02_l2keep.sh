for mb in 0 32 64 96; do
  echo "keep_mb=$mb"
  F2M_L2_KEEP_MB=$mb timeout 900 python tools/ab_sweep.py exp/prevstream . --n 2000000 --sweeps 300 --reps 2 < /dev/null 2>&1 | cut -c1-120
done
F2M_L2_KEEP_MB=64 timeout 900 python tools/ab_sweep.py exp/prevstream . --n 1000000 --sweeps 600 --reps 2 < /dev/null 2>&1 | cut -c1-120
F2M_L2_KEEP_MB=64 timeout 900 python tools/ab_sweep.py exp/prevstream . --n 400000 --sweeps 1000 --reps 2 < /dev/null 2>&1 | cut -c1-120

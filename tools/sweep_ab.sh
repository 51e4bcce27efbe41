#!/bin/bash
# A/B of sweep-kernel variants / knobs: us per sweep at 10k / 100k / 200k (2000 sweeps each),
# configurations interleaved over REPS rounds (box-to-box and run-to-run noise is ~10%).
REPS=${REPS:-2}
for r in $(seq 1 $REPS); do
  for cfg in "$@"; do
    for n in 10000 100000 200000; do
      echo "$cfg n=$n $(env $cfg timeout 120 python tools/profile_sweep.py $n 2000 2>&1 | grep us/sweep | sed 's/.*us\/sweep=\([0-9.]*\).*/\1/')"
    done
  done
done

mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base exp/norescan . --n 100000 --sweeps 3000 --reps 3 < /dev/null > gpurun_out/head4.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base exp/norescan . --n 200000 --sweeps 3000 --reps 2 < /dev/null >> gpurun_out/head4.log 2>&1
cat gpurun_out/head4.log

mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base exp/lane . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/ab35.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base exp/lane . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/ab35.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base . --n 200000 --solve --clustered --reps 2 < /dev/null >> gpurun_out/ab35.log 2>&1
cut -c1-130 gpurun_out/ab35.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest35.log 2>&1; echo "rc=$?" >> gpurun_out/pytest35.log; tail -2 gpurun_out/pytest35.log

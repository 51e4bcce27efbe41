mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest31.log 2>&1; echo "rc=$?" >> gpurun_out/pytest31.log
tail -3 gpurun_out/pytest31.log
timeout 600 python tools/ab_sweep.py exp/base . exp/base . --n 100000 --sweeps 3000 --reps 2 < /dev/null > gpurun_out/ab31.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base . --n 100000 --solve --reps 3 < /dev/null >> gpurun_out/ab31.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/ab31.log 2>&1
cat gpurun_out/ab31.log

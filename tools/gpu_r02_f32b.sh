mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/head64 . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/f32b.log 2>&1
timeout 900 python tools/ab_sweep.py exp/head64 . --n 50000 --solve --reps 2 < /dev/null >> gpurun_out/f32b.log 2>&1
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest_f32b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f32b.log
cat gpurun_out/f32b.log; tail -3 gpurun_out/pytest_f32b.log

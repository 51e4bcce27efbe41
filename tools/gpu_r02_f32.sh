mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/head64 . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/f32.log 2>&1
timeout 900 python tools/ab_sweep.py exp/head64 . --n 50000 --solve --reps 3 < /dev/null >> gpurun_out/f32.log 2>&1
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py tests/test_gpu_primal.py tests/test_gpu_multi_gpu.py tests/test_sharded.py < /dev/null > gpurun_out/pytest_f32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f32.log
cat gpurun_out/f32.log; tail -15 gpurun_out/pytest_f32.log

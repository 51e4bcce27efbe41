mkdir -p gpurun_out
timeout 900 python tools/ab_stages.py exp/base . exp/base . --n 100000 < /dev/null > gpurun_out/ab18.log 2>&1
timeout 900 python tools/ab_stages.py exp/base . --n 200000 --reps 7 < /dev/null >> gpurun_out/ab18.log 2>&1
timeout 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_primal.py tests/test_gpu_headline.py tests/test_gpu_reference_unit_suite.py < /dev/null > gpurun_out/pytest18.log 2>&1; echo "rc=$?" >> gpurun_out/pytest18.log
cat gpurun_out/ab18.log; tail -3 gpurun_out/pytest18.log

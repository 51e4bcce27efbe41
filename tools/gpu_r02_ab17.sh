mkdir -p gpurun_out
timeout 900 python tools/ab_stages.py exp/base . exp/base . --n 100000 < /dev/null > gpurun_out/ab17.log 2>&1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_knn.py tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest17.log 2>&1; echo "rc=$?" >> gpurun_out/pytest17.log
cat gpurun_out/ab17.log; tail -2 gpurun_out/pytest17.log

mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 200000 --clustered --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1
timeout 900 python tools/ab_sweep.py exp/nolayout . --n 10000 --solve --reps 2 < /dev/null >> gpurun_out/bank.log 2>&1
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py tests/test_gpu_primal.py < /dev/null > gpurun_out/pytest_bank.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bank.log
cut -c1-120 gpurun_out/bank.log; tail -3 gpurun_out/pytest_bank.log

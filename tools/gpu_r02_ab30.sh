mkdir -p gpurun_out
timeout 600 python tools/ab_sweep.py exp/base . exp/base . --n 100000 --sweeps 3000 --reps 3 < /dev/null > gpurun_out/ab30.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base . --n 200000 --sweeps 2000 --reps 3 < /dev/null >> gpurun_out/ab30.log 2>&1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py < /dev/null > gpurun_out/pytest30.log 2>&1; echo "rc=$?" >> gpurun_out/pytest30.log
cat gpurun_out/ab30.log; tail -3 gpurun_out/pytest30.log

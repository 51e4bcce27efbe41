mkdir -p gpurun_out
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_multi_gpu.py < /dev/null > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
timeout 900 python tools/ab_sweep.py . exp/st768 --n 2000000 --sweeps 300 --reps 2 --inner 2 < /dev/null > gpurun_out/ab_st768.log 2>&1
bash tools/gpu_r02_profile.sh
tail -2 gpurun_out/pytest_multi.log; cat gpurun_out/ab_st768.log

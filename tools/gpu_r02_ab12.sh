mkdir -p gpurun_out
for n in 100000 200000 10000 1000; do
  timeout 900 python tools/ab_sweep.py exp/base . --n $n --solve --reps 2 --inner 3 < /dev/null
done > gpurun_out/ab12.log 2>&1
timeout 300 python tools/ab_sweep.py exp/base . --n 200000 --clustered --solve --reps 2 --inner 3 < /dev/null >> gpurun_out/ab12.log 2>&1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_dual.py tests/test_gpu_headline.py < /dev/null > gpurun_out/pytest12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest12.log
cat gpurun_out/ab12.log; tail -3 gpurun_out/pytest12.log

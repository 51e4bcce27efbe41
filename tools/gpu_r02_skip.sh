# tail skipping: A/B against the build without it, GPU suite, smoke, bench, configs, ncu of the 100k sweep
mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base . exp/base . --n 100000 --solve --reps 2 < /dev/null > gpurun_out/ab_skip.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/ab_skip.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 200000 --clustered --solve --reps 2 < /dev/null >> gpurun_out/ab_skip.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 10000 --solve --reps 2 < /dev/null >> gpurun_out/ab_skip.log 2>&1
cut -c1-120 gpurun_out/ab_skip.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider < /dev/null > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" < /dev/null > gpurun_out/smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke.log
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
timeout 900 python tools/configs_run.py < /dev/null > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gdp_sweep5 -c 1 -f \
   -o gpurun_out/r02s_sweep100k python tools/profile_sweep.py 100000 3000 < /dev/null > gpurun_out/ncu_s100k.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log

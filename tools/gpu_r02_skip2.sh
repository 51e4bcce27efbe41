# tail skipping gated off in the small-graph (PAIR) form: A/B at 10k and 100k, GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base . --n 10000 --solve --reps 3 < /dev/null > gpurun_out/ab_skip2.log 2>&1
timeout 900 python tools/ab_sweep.py exp/base . --n 100000 --solve --reps 2 < /dev/null >> gpurun_out/ab_skip2.log 2>&1
cut -c1-120 gpurun_out/ab_skip2.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider < /dev/null > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" < /dev/null > gpurun_out/smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke.log
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
timeout 900 python tools/configs_run.py < /dev/null > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --no-extra < /dev/null > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log

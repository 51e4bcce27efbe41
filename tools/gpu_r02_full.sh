# full GPU test suite + smoke + default bench (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider < /dev/null > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" < /dev/null > gpurun_out/smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke.log
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --steps 20 --warmup 5 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log

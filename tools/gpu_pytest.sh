# full GPU test suite + smoke (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider < /dev/null > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" < /dev/null > gpurun_out/smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log

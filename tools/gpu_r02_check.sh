# round-2 GPU check: new GPU tests, tput microbench, one bench run (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_instance.py tests/test_gpu_multi_gpu.py \
  tests/test_gpu_cpp_api.py tests/test_gpu_reference_unit_suite.py tests/test_gpu_2m.py > gpurun_out/pytest_new.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_new.log
./oracle/_ref/b200_binding/f2m_refsuite > gpurun_out/refsuite.log 2>&1; echo "refsuite_rc=$?" >> gpurun_out/refsuite.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench/tput.cu -o /tmp/tput && timeout 120 /tmp/tput > gpurun_out/tput.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench/latency.cu -o /tmp/lat && timeout 60 /tmp/lat > gpurun_out/latency.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench/rowlat.cu -o /tmp/rowlat && timeout 60 /tmp/rowlat > gpurun_out/rowlat.log 2>&1
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
tail -3 gpurun_out/pytest_new.log

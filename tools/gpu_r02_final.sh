# round-2 evidence run: GPU suite, smoke, bench (driver's arguments), reference arm, every config,
# ncu launch list of the bench, ncu captures of the final sweep kernels (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider < /dev/null > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" < /dev/null > gpurun_out/smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke.log
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
timeout 900 python tools/configs_run.py < /dev/null > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --no-extra < /dev/null > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gdp_sweep5 -c 1 -f \
   -o gpurun_out/r02f_sweep2m python tools/profile_sweep.py 2000000 64 < /dev/null > gpurun_out/ncu_f2m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gdp_sweep5 -c 1 -f \
   -o gpurun_out/r02f_sweep100k python tools/profile_sweep.py 100000 3000 < /dev/null > gpurun_out/ncu_f100k.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:allpairs_sweep -c 1 -f \
   -o gpurun_out/r02f_ap8000dense python tools/profile_sweep.py 8000 20 allpairs < /dev/null > gpurun_out/ncu_fap.log 2>&1
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
echo "ref_rc=$?"
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; ls gpurun_out

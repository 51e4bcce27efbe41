mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py exp/base exp/nob . --n 100000 --solve --reps 3 < /dev/null > gpurun_out/ab36.log 2>&1
timeout 600 python tools/ab_sweep.py exp/base exp/nob . --n 200000 --solve --reps 2 < /dev/null >> gpurun_out/ab36.log 2>&1
cut -c1-110 gpurun_out/ab36.log
for v in wprof0 wprof1 wprofn; do timeout 300 python tools/sweep_trace.py exp/$v < /dev/null 2>&1 | tail -1 >> gpurun_out/trace36.log; timeout 300 python tools/warp_profile.py exp/$v < /dev/null 2>&1 | tail -1 | cut -c1-700 >> gpurun_out/trace36.log; done
cat gpurun_out/trace36.log

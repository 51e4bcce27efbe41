mkdir -p gpurun_out
for v in wprof0 wprof1; do timeout 300 python tools/warp_profile.py exp/$v < /dev/null 2>&1 | tail -1 >> gpurun_out/wprof34.log; done
cat gpurun_out/wprof34.log

mkdir -p gpurun_out
timeout 900 python tools/ab_stages.py exp/base . exp/base . --n 100000 < /dev/null > gpurun_out/ab14.log 2>&1
cat gpurun_out/ab14.log

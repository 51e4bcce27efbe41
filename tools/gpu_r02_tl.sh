mkdir -p gpurun_out
timeout 300 python tools/timeline.py 100000 < /dev/null > gpurun_out/timeline.txt 2>&1
head -120 gpurun_out/timeline.txt

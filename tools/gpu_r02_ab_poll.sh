mkdir -p gpurun_out
timeout 900 python tools/ab_sweep.py . exp/poll32 exp/poll128 exp/poll256 --n 100000 --solve --reps 3 --inner 3 < /dev/null > gpurun_out/ab_poll_100k.log 2>&1
timeout 900 python tools/ab_sweep.py . exp/poll32 exp/poll128 exp/poll256 --n 200000 --solve --reps 2 --inner 3 < /dev/null > gpurun_out/ab_poll_200k.log 2>&1
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1200 python bench.py --steps 5 --warmup 3 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo bench_rc=$?
cat gpurun_out/ab_poll_100k.log gpurun_out/ab_poll_200k.log

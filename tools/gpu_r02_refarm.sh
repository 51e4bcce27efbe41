mkdir -p gpurun_out
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
echo "ref_rc=$?"
TORCH_SYMM_MEM_DISABLE_MULTICAST=1 timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 < /dev/null > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench_rc=$?"
tail -c 600 gpurun_out/bench_ref.jsonl

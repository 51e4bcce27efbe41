# round-2 ncu captures (one launch each, --set full) + un-profiled timings of the same commands
mkdir -p gpurun_out
for spec in "8000 20 allpairs:allpairs_sweep:ap8000" "2000 200 allpairs:allpairs_sweep:ap2000" \
            "2000000 64 x:gdp_sweep5:sweep2m" "100000 300 x:gdp_sweep5:sweep100k"; do
  args=${spec%%:*}; rest=${spec#*:}; kre=${rest%%:*}; name=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -f \
    -o gpurun_out/r02_$name python tools/profile_sweep.py $args > gpurun_out/ncu_$name.log 2>&1 < /dev/null
  echo "$name ncu_rc=$?"
  timeout 300 python tools/profile_sweep.py $args > gpurun_out/time_$name.log 2>&1 < /dev/null
done
python tools/ncu_summarize.py gpurun_out/r02_*.ncu-rep > gpurun_out/r02_ncu_summary.jsonl 2>&1 < /dev/null
ls -la gpurun_out

set -x
mkdir -p gpurun_out
./oracle/_ref/b200_binding/f2m_refsuite > gpurun_out/refsuite.log 2>&1; echo refsuite_rc=$? >> gpurun_out/refsuite.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench/tput.cu -o /tmp/tput && /tmp/tput > gpurun_out/tput.log 2>&1
for spec in "8000 20 allpairs:allpairs_sweep:ap8000" "2000 200 allpairs:allpairs_sweep:ap2000" "2000000 64 x:gdp_sweep5:sweep2m" "100000 300 x:gdp_sweep5:sweep100k"; do
  args=${spec%%:*}; rest=${spec#*:}; kre=${rest%%:*}; name=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -f -o gpurun_out/r02_$name python tools/profile_sweep.py $args > gpurun_out/ncu_$name.log 2>&1
  python tools/profile_sweep.py $args > gpurun_out/time_$name.log 2>&1
done
ls -la gpurun_out

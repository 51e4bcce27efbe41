mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_dual.py -k allpairs < /dev/null > gpurun_out/pytest_ap.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ap.log
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.allpairs_leg(None)))
" < /dev/null > gpurun_out/ap_leg.json 2>&1
tail -2 gpurun_out/pytest_ap.log; cat gpurun_out/ap_leg.json | head -c 3000

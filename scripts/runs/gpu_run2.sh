timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -s -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python scripts/tc_perf.py 5 10 > gpurun_out/tc_perf_c5.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_perf_c5.txt
timeout 300 python scripts/tc_perf.py 3 10 > gpurun_out/tc_perf_c3.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_perf_c3.txt
timeout 300 python scripts/tc_perf.py 2 50 > gpurun_out/tc_perf_c2.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_perf_c2.txt

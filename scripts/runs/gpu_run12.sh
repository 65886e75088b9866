timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python scripts/tc_perf.py 3 10 tc,ffma > gpurun_out/tc_perf_c3.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_perf_c3.txt
timeout 300 python scripts/trace_tc.py 3 > gpurun_out/trace_tc_c3.txt 2>&1; echo "rc=$?" >> gpurun_out/trace_tc_c3.txt
timeout 300 python scripts/tc_perf.py 5 10 tc > gpurun_out/tc_perf_c5.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_perf_c5.txt

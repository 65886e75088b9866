timeout 300 python scripts/tc_perf.py 6 5 ffma > gpurun_out/perf_c6.txt 2>&1; echo "rc=$?" >> gpurun_out/perf_c6.txt
HSNCT_NO_PERSIST=1 timeout 300 python scripts/tc_perf.py 6 5 ffma >> gpurun_out/perf_c6.txt 2>&1; echo "rc=$?" >> gpurun_out/perf_c6.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "nmf or clamped" > gpurun_out/pytest_k12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k12.log

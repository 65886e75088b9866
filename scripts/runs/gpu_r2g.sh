timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_fulliter.py -x -q -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest.log
timeout 300 python scripts/tc_perf.py 6 10 mma > gpurun_out/r2g_c6.txt 2>&1
timeout 300 python scripts/tc_perf.py 5 10 mma > gpurun_out/r2g_c5.txt 2>&1

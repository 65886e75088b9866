timeout 1200 python -m pytest tests/test_gpu_mma.py tests/test_gpu_counts.py tests/test_gpu_fulliter.py -x -q -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
timeout 300 python scripts/tc_perf.py 5 10 mma > gpurun_out/r2i_c5.txt 2>&1
timeout 300 python scripts/counts_perf.py > gpurun_out/r2i_counts.txt 2>&1

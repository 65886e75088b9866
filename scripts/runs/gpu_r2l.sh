timeout 900 python -m pytest tests/test_gpu_counts.py tests/test_gpu_mma.py -x -q -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.log
timeout 300 python scripts/counts_perf.py 3 > gpurun_out/r2l_counts3.txt 2>&1
timeout 300 python scripts/counts_perf.py 5 > gpurun_out/r2l_counts5.txt 2>&1

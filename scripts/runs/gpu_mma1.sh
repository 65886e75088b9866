timeout 600 python -m pytest tests/test_gpu_mma.py -x -q -p no:cacheprovider > gpurun_out/mma1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mma1_pytest.log
timeout 300 python scripts/tc_perf.py 3 10 mma,ffma > gpurun_out/mma1_perf_c3.txt 2>&1
timeout 300 python scripts/tc_perf.py 5 10 mma,ffma > gpurun_out/mma1_perf_c5.txt 2>&1
timeout 300 python scripts/tc_perf.py 2 50 mma,ffma > gpurun_out/mma1_perf_c2.txt 2>&1

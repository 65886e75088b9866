timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/tc_perf.py 6 5 ffma > gpurun_out/perf_c6.txt 2>&1; echo "rc=$?" >> gpurun_out/perf_c6.txt

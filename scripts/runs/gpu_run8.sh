timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nmf_tc -c 1 -f -o gpurun_out/ncu_tc2_c3 python scripts/tc_perf.py 3 2 tc > gpurun_out/ncu_tc2.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_tc2.log

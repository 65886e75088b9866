timeout 600 python -m pytest tests/test_gpu_mma.py -x -q -p no:cacheprovider > gpurun_out/mma3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mma3_pytest.log
timeout 300 python scripts/tc_perf.py 3 10 mma,ffma > gpurun_out/mma3_perf_c3.txt 2>&1
timeout 300 python scripts/tc_perf.py 5 10 mma,ffma > gpurun_out/mma3_perf_c5.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 2 -c 1 -o gpurun_out/ncu_mma3_c3 python scripts/tc_perf.py 3 4 mma > gpurun_out/ncu_mma3_c3.log 2>&1

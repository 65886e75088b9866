L=$PWD/paper_2410_22500_b200/libhsnct_nodistv.so
timeout 1200 python -m pytest tests/test_gpu_mma.py tests/test_gpu_counts.py tests/test_gpu_fulliter.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_pytest.log
for i in 1 2; do
HSNCT_LIB=$L timeout 300 python scripts/tc_perf.py 6 30 mma >> gpurun_out/r2p_ab6.txt 2>&1
timeout 300 python scripts/tc_perf.py 6 30 mma >> gpurun_out/r2p_ab6.txt 2>&1
done

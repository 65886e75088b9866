L=$PWD/paper_2410_22500_b200/libhsnct_distv.so
HSNCT_LIB=$L timeout 600 python -m pytest tests/test_gpu_mma.py -x -q -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_pytest.log
for i in 1 2; do
HSNCT_LIB=$L timeout 300 python scripts/tc_perf.py 5 40 mma >> gpurun_out/r2o_ab.txt 2>&1
timeout 300 python scripts/tc_perf.py 5 40 mma >> gpurun_out/r2o_ab.txt 2>&1
done

for i in 1 2; do
HSNCT_LIB=$PWD/paper_2410_22500_b200/libhsnct_old.so timeout 300 python scripts/tc_perf.py 5 20 mma >> gpurun_out/r2j_ab.txt 2>&1
timeout 300 python scripts/tc_perf.py 5 20 mma >> gpurun_out/r2j_ab.txt 2>&1
done

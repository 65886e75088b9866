HSNCT_LIB=$PWD/paper_2410_22500_b200/libhsnct_old.so ncu --set full --clock-control none -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/ab_old python scripts/tc_perf.py 5 3 mma > gpurun_out/ab_old.log 2>&1
ncu --set full --clock-control none -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/ab_new python scripts/tc_perf.py 5 3 mma > gpurun_out/ab_new.log 2>&1

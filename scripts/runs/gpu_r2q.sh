ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/ncu_mma_c5_v5 python scripts/tc_perf.py 5 3 mma > gpurun_out/ncu_mma_c5_v5.log 2>&1

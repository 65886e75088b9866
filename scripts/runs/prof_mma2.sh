ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 2 -c 1 -o gpurun_out/ncu_mma_c3 python scripts/tc_perf.py 3 4 mma > gpurun_out/ncu_mma_c3.log 2>&1
echo rc=$?

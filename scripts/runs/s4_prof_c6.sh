# session 4: ncu --set full of the final C6 kernel (packed second column block, skipped dummy block)
mkdir -p gpurun_out/s4
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/s4/ncu_mma_c6_final python scripts/tc_perf.py 6 3 mma > gpurun_out/s4/ncu_mma_c6_final.log 2>&1; echo "ncu c6 rc=$?"

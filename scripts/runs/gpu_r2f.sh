B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dhr --no-fmd --no-mbir --no-counts"
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:"^k_" -c 400 --csv --log-file gpurun_out/r2f_launches_c5.csv $B > gpurun_out/r2f_ncu.log 2>&1
echo rc=$? >> gpurun_out/r2f_ncu.log
ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/ncu_mma_c6 python scripts/tc_perf.py 6 3 mma > gpurun_out/ncu_mma_c6.log 2>&1

# session 4: launch list of the default bench step and ncu --set full of the final mma pass (C5 and C6), after the bench exits 0 without ncu
mkdir -p gpurun_out/s4
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dhr --no-fmd --no-mbir --no-counts"
timeout 600 $B > gpurun_out/s4/bench_c5_short.json 2> gpurun_out/s4/bench_c5_short.err; echo "bench rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:"^k_" -c 400 --csv --log-file gpurun_out/s4/launches_c5.csv $B > gpurun_out/s4/launches_ncu.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/s4/ncu_mma_c5_s4 python scripts/tc_perf.py 5 3 mma > gpurun_out/s4/ncu_mma_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/s4/ncu_mma_c6_s4 python scripts/tc_perf.py 6 3 mma > gpurun_out/s4/ncu_mma_c6.log 2>&1; echo "ncu c6 rc=$?"
ls -la gpurun_out/s4/

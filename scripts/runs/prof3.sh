B="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 4 --no-e2e --no-cpu --no-dhr"
$B > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_fused|k_dred|k_yplus" -s 1 -c 3 -o gpurun_out/prof_fused2 $B > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu4.log
B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 10 --no-e2e --no-cpu --no-dhr"
$B2 > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_c2.csv $B2 > gpurun_out/ncu5.log 2>&1
tail -1 gpurun_out/ncu5.log

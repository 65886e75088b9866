B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 10 --no-e2e --no-cpu --no-dhr"
$B2 > gpurun_out/plain_m2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_mma" -s 1 -c 1 -o gpurun_out/prof_mma_c2 $B2 > gpurun_out/ncu_m2.log 2>&1
echo rc=$?

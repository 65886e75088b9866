# FMD kernels at C4 (NNLS is the big one): plain run, then ncu --set full of the FMD launches
B4="python bench.py --config 4 --steps 1 --warmup 1 --n-iter 2 --no-e2e --no-cpu --no-dhr"
$B4 > gpurun_out/plain_fmd4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fmd" -c 6 -o gpurun_out/prof_fmd4 $B4 > gpurun_out/ncu_fmd4.log 2>&1
echo "fmd rc=$?"

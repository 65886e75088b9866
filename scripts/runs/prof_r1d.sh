# source-level capture of the C2 NMF kernel (instruction hot spots)
B2="python bench.py --config 2 --steps 1 --warmup 1 --n-iter 20 --no-e2e --no-cpu --no-dhr --no-fmd"
$B2 > gpurun_out/plain_c2g.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nmf_persist" -s 1 -c 1 -o gpurun_out/prof_c2g $B2 > gpurun_out/ncu_c2g.log 2>&1
echo "c2 rc=$?"
ls -la gpurun_out/
